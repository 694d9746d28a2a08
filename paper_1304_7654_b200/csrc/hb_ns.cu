// hb_ns.cu -- the north-star HB Euler / laminar Navier-Stokes stage (SURVEY.md
// §8 row f2), specified in nsflow.py's docstring: central convective flux
// with JST artificial dissipation (2-cell halos), laminar viscous flux on a
// face "diamond", curvilinear metrics with optional rigid grid motion,
// far-field / no-slip / slip-wall / cut halos, local time stepping, the HB
// source V D W, 4-stage RK.  The reference has no such physics; parity is
// against the builder-written oracle/ns_oracle.c (unpinned), bitwise.
//
// Layout: one pool per state slot holding every block, block b's value
// (n, k, j, i) -- i, j in [-1, n+2] -- at w_off + ((n*4 + k)*(nj+4) + j+1)*(ni+4)
// + i+1; the residual pool (P, 4, nj, ni) per block; geometry pools as
// nsflow.metrics (geometry snapshot g = n when the mesh moves, else 0).
//
// Kernels (all strict IEEE mul/add/div/sqrt in the specification's order):
//   ns_bc_kernel        non-cut sides' two halo layers, one thread per
//                       (side, layer, face cell, snapshot)
//   ns_corner_kernel    corner halos
//   ns_timestep_kernel  local time step, one thread per cell
//   ns_prim_kernel      u, v, p, c, e of every cell (halos included) once per
//                       stage: the flux kernel reads each cell's up to 20 times
//   ns_residual_kernel  face fluxes -> R, one thread per (cell, snapshot)
//   ns_update_kernel    HB source + RK update, one thread per (cell,
//                       variable) for all snapshots; stage-1 R_rho^2 partials
//                       per CTA, folded by ns_norm_kernel (a warp per block)
//   ns_forces_kernel    wall pressure forces, one thread per snapshot
// Cut halos move with hbgpu_halo (two directions per cut and layer).

#include "hb_common.cuh"

#include "hbns.h"

namespace hbns {

constexpr double GAMMA = 1.4;
constexpr double PR = 0.72;
constexpr double K2 = 0.5;
constexpr double K4 = 1.0 / 64.0;
constexpr int NV = 4;

__device__ __forceinline__ int64_t ws(const hbns_block &b, int n, int k, int j, int i) {
    return b.w_off + (((int64_t)n * NV + k) * (b.nj + 4) + (j + 1)) * (b.ni + 4) + (i + 1);
}
__device__ __forceinline__ int64_t rs(const hbns_block &b, int n, int k, int j, int i) {
    return b.r_off + (((int64_t)n * NV + k) * b.nj + (j - 1)) * b.ni + (i - 1);
}
__device__ __forceinline__ int64_t cc(const hbns_block &b, int g, int j, int i) {
    return b.c_off + ((int64_t)g * (b.nj + 4) + (j + 1)) * (b.ni + 4) + (i + 1);
}
__device__ __forceinline__ int64_t fi(const hbns_block &b, int g, int j, int i) {
    return b.fi_off + ((int64_t)g * (b.nj + 4) + (j + 1)) * (b.ni + 5) + (i + 2);
}
__device__ __forceinline__ int64_t fj(const hbns_block &b, int g, int j, int i) {
    return b.fj_off + ((int64_t)g * (b.nj + 5) + (j + 2)) * (b.ni + 4) + (i + 1);
}

struct Prim {
    double r, ru, rv, re, u, v, p, c, e;
};

// the primitive pool (u, v, p, c, e) of every cell of a slot, halos included
constexpr int NPRIM = 5;
__device__ __forceinline__ int64_t ps_(const hbns_block &b, int n, int k, int j, int i) {
    return b.w_off / NV * NPRIM + (((int64_t)n * NPRIM + k) * (b.nj + 4) + (j + 1)) * (b.ni + 4) + (i + 1);
}

__device__ __forceinline__ Prim prim(const double *w, int64_t stride) {
    Prim q;
    q.r = w[0];
    q.ru = w[stride];
    q.rv = w[2 * stride];
    q.re = w[3 * stride];
    q.u = __ddiv_rn(q.ru, q.r);
    q.v = __ddiv_rn(q.rv, q.r);
    q.p = __dmul_rn(GAMMA - 1.0, __dsub_rn(q.re, __dmul_rn(0.5, __dadd_rn(__dmul_rn(q.ru, q.u), __dmul_rn(q.rv, q.v)))));
    q.c = __dsqrt_rn(__ddiv_rn(__dmul_rn(GAMMA, q.p), q.r));
    q.e = __ddiv_rn(q.p, __dmul_rn(GAMMA - 1.0, q.r));
    return q;
}

__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dv(double a, double b) { return __ddiv_rn(a, b); }

// ---- halos --------------------------------------------------------------------------------

__global__ void ns_bc_kernel(hbns_args a, double *w) {
    // grid.y = block, grid.z = snapshot; x: (side, layer, face cell) flattened
    const hbns_block &b = a.blocks[blockIdx.y];
    const int n = blockIdx.z;
    const int g = a.Pg > 1 ? n : 0;
    const int maxlen = b.ni > b.nj ? b.ni : b.nj;
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= 8 * maxlen) return;
    const int side = t / (2 * maxlen);
    const int layer = (t / maxlen) % 2 + 1;
    const int e = t % maxlen + 1;
    const int kind = b.kinds[side];
    const int len = side < 2 ? b.ni : b.nj;
    if (kind == HBNS_CUT || e > len) return;
    int hi_, hj, ii, ij;
    int64_t f;
    const double *sxa, *sya, *ga;
    if (side == 0) {
        hi_ = e; hj = 1 - layer; ii = e; ij = layer;
        f = fj(b, g, 0, e); sxa = a.sjx; sya = a.sjy; ga = a.gj;
    } else if (side == 1) {
        hi_ = e; hj = b.nj + layer; ii = e; ij = b.nj + 1 - layer;
        f = fj(b, g, b.nj, e); sxa = a.sjx; sya = a.sjy; ga = a.gj;
    } else if (side == 2) {
        hi_ = 1 - layer; hj = e; ii = layer; ij = e;
        f = fi(b, g, e, 0); sxa = a.six; sya = a.siy; ga = a.gi;
    } else {
        hi_ = b.ni + layer; hj = e; ii = b.ni + 1 - layer; ij = e;
        f = fi(b, g, e, b.ni); sxa = a.six; sya = a.siy; ga = a.gi;
    }
    const int64_t st = (int64_t)(b.nj + 4) * (b.ni + 4);
    double out[NV];
    if (kind == HBNS_FARFIELD) {
        for (int k = 0; k < NV; ++k) out[k] = a.winf[NV * n + k];
    } else {
        const Prim q = prim(w + ws(b, n, 0, ij, ii), st);
        if (kind == HBNS_NOSLIP) {
            out[0] = q.r;
            out[1] = -q.ru;
            out[2] = -q.rv;
            out[3] = q.re;
        } else {
            const double sx = sxa[f], sy = sya[f];
            const double gg = a.moving ? ga[f] : 0.0;
            const double sa = __dsqrt_rn(add(mul(sx, sx), mul(sy, sy)));
            const double nx = dv(sx, sa), ny = dv(sy, sa);
            const double vn = sub(add(mul(q.u, nx), mul(q.v, ny)), dv(gg, sa));
            const double ug = sub(q.u, mul(mul(2.0, vn), nx));
            const double vg = sub(q.v, mul(mul(2.0, vn), ny));
            out[0] = q.r;
            out[1] = mul(q.r, ug);
            out[2] = mul(q.r, vg);
            out[3] = add(dv(q.p, GAMMA - 1.0), mul(mul(0.5, q.r), add(mul(ug, ug), mul(vg, vg))));
        }
    }
    for (int k = 0; k < NV; ++k) w[ws(b, n, k, hj, hi_)] = out[k];
}

__global__ void ns_corner_kernel(hbns_args a, double *w) {
    // grid.y = block, grid.z = snapshot * 4 + variable; x: the 4 halo columns
    // x 4 corner rows
    const hbns_block &b = a.blocks[blockIdx.y];
    const int n = blockIdx.z / NV, k = blockIdx.z % NV;
    const int t = threadIdx.x;
    if (t >= 16) return;
    const int col = t % 4, row = t / 4;
    const int i = col < 2 ? col - 1 : b.ni + col - 1;       // -1, 0, ni+1, ni+2
    const int j = row < 2 ? row - 1 : b.nj + row - 1;       // -1, 0, nj+1, nj+2
    const int src = row < 2 ? 1 : b.nj;
    w[ws(b, n, k, j, i)] = w[ws(b, n, k, src, i)];
}

// ---- primitives: one conversion per cell and stage (the flux kernel reads
// each cell's u, v, p, c, e up to 20 times) -----------------------------------------------

__global__ void ns_prim_kernel(hbns_args a, const double *w) {
    // grid.y = block, grid.z = snapshot; x over all cells incl. the halo ring
    const hbns_block &b = a.blocks[blockIdx.y];
    const int n = blockIdx.z;
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    const int wi = b.ni + 4;
    if (t >= wi * (b.nj + 4)) return;
    const int i = t % wi - 1, j = t / wi - 1;
    const int64_t st = (int64_t)(b.nj + 4) * (b.ni + 4);
    const Prim q = prim(w + ws(b, n, 0, j, i), st);
    a.prim[ps_(b, n, 0, j, i)] = q.u;
    a.prim[ps_(b, n, 1, j, i)] = q.v;
    a.prim[ps_(b, n, 2, j, i)] = q.p;
    a.prim[ps_(b, n, 3, j, i)] = q.c;
    a.prim[ps_(b, n, 4, j, i)] = q.e;
}

// a cell's state and primitives, the latter from the pool
__device__ __forceinline__ Prim load_prim(const hbns_args &a, const hbns_block &b, const double *w, int n, int j,
                                          int i) {
    const int64_t st = (int64_t)(b.nj + 4) * (b.ni + 4);
    const double *c = w + ws(b, n, 0, j, i);
    Prim q;
    q.r = c[0];
    q.ru = c[st];
    q.rv = c[2 * st];
    q.re = c[3 * st];
    q.u = a.prim[ps_(b, n, 0, j, i)];
    q.v = a.prim[ps_(b, n, 1, j, i)];
    q.p = a.prim[ps_(b, n, 2, j, i)];
    q.c = a.prim[ps_(b, n, 3, j, i)];
    q.e = a.prim[ps_(b, n, 4, j, i)];
    return q;
}

// ---- fluxes -----------------------------------------------------------------------------

__device__ void face_flux(const hbns_args &a, const hbns_block &b, const double *w, int n, int g, int jL, int iL,
                          int dj, int di, double sx, double sy, double gf, double *out) {
    const int jR = jL + dj, iR = iL + di;
    const Prim L = load_prim(a, b, w, n, jL, iL), R = load_prim(a, b, w, n, jR, iR);
    const Prim LL = load_prim(a, b, w, n, jL - dj, iL - di);
    const Prim RR = load_prim(a, b, w, n, jR + dj, iR + di);
    const double unL = add(mul(L.u, sx), mul(L.v, sy)), unR = add(mul(R.u, sx), mul(R.v, sy));
    const double urL = sub(unL, gf), urR = sub(unR, gf);
    double FL[NV] = {mul(L.r, urL), add(mul(L.ru, urL), mul(L.p, sx)), add(mul(L.rv, urL), mul(L.p, sy)),
                     add(mul(L.re, urL), mul(L.p, unL))};
    double FR[NV] = {mul(R.r, urR), add(mul(R.ru, urR), mul(R.p, sx)), add(mul(R.rv, urR), mul(R.p, sy)),
                     add(mul(R.re, urR), mul(R.p, unR))};
    const double sa = __dsqrt_rn(add(mul(sx, sx), mul(sy, sy)));
    const double lamL = add(fabs(urL), mul(L.c, sa)), lamR = add(fabs(urR), mul(R.c, sa));
    const double lam = mul(0.5, add(lamL, lamR));
    const double nuL = dv(fabs(add(sub(R.p, mul(2.0, L.p)), LL.p)), add(add(R.p, mul(2.0, L.p)), LL.p));
    const double nuR = dv(fabs(add(sub(RR.p, mul(2.0, R.p)), L.p)), add(add(RR.p, mul(2.0, R.p)), L.p));
    const double eps2 = mul(mul(K2, lam), fmax(nuL, nuR));
    const double eps4 = fmax(0.0, sub(mul(K4, lam), eps2));
    double fv[NV] = {0.0, 0.0, 0.0, 0.0};
    const bool visc = a.mu > 0.0;
    if (visc) {
        const int tj = di, ti = dj;
        const Prim Lp = load_prim(a, b, w, n, jL + tj, iL + ti), Rp = load_prim(a, b, w, n, jR + tj, iR + ti);
        const Prim Lm = load_prim(a, b, w, n, jL - tj, iL - ti), Rm = load_prim(a, b, w, n, jR - tj, iR - ti);
        const double xL = a.xc[cc(b, g, jL, iL)], xR = a.xc[cc(b, g, jR, iR)];
        const double yL = a.yc[cc(b, g, jL, iL)], yR = a.yc[cc(b, g, jR, iR)];
        const double xLp = a.xc[cc(b, g, jL + tj, iL + ti)], xRp = a.xc[cc(b, g, jR + tj, iR + ti)];
        const double xLm = a.xc[cc(b, g, jL - tj, iL - ti)], xRm = a.xc[cc(b, g, jR - tj, iR - ti)];
        const double yLp = a.yc[cc(b, g, jL + tj, iL + ti)], yRp = a.yc[cc(b, g, jR + tj, iR + ti)];
        const double yLm = a.yc[cc(b, g, jL - tj, iL - ti)], yRm = a.yc[cc(b, g, jR - tj, iR - ti)];
        const double x_a = sub(xR, xL), y_a = sub(yR, yL);
        const double x_b = mul(0.25, sub(add(xLp, xRp), add(xLm, xRm)));
        const double y_b = mul(0.25, sub(add(yLp, yRp), add(yLm, yRm)));
        const double jac = sub(mul(x_a, y_b), mul(x_b, y_a));
        const double ua = sub(R.u, L.u), ub = mul(0.25, sub(add(Lp.u, Rp.u), add(Lm.u, Rm.u)));
        const double va = sub(R.v, L.v), vb = mul(0.25, sub(add(Lp.v, Rp.v), add(Lm.v, Rm.v)));
        const double ea = sub(R.e, L.e), eb = mul(0.25, sub(add(Lp.e, Rp.e), add(Lm.e, Rm.e)));
        const double ux = dv(sub(mul(ua, y_b), mul(ub, y_a)), jac), uy = dv(sub(mul(ub, x_a), mul(ua, x_b)), jac);
        const double vx = dv(sub(mul(va, y_b), mul(vb, y_a)), jac), vy = dv(sub(mul(vb, x_a), mul(va, x_b)), jac);
        const double ex = dv(sub(mul(ea, y_b), mul(eb, y_a)), jac), ey = dv(sub(mul(eb, x_a), mul(ea, x_b)), jac);
        const double mu = a.mu;
        const double div = add(ux, vy);
        const double t23 = 2.0 / 3.0;
        const double txx = mul(mu, sub(mul(2.0, ux), mul(t23, div)));
        const double tyy = mul(mu, sub(mul(2.0, vy), mul(t23, div)));
        const double txy = mul(mu, add(uy, vx));
        const double kq = dv(mul(mu, GAMMA), PR);
        const double qx = -mul(kq, ex), qy = -mul(kq, ey);
        const double uf = mul(0.5, add(L.u, R.u)), vf = mul(0.5, add(L.v, R.v));
        fv[1] = add(mul(txx, sx), mul(txy, sy));
        fv[2] = add(mul(txy, sx), mul(tyy, sy));
        fv[3] = add(mul(sub(add(mul(uf, txx), mul(vf, txy)), qx), sx), mul(sub(add(mul(uf, txy), mul(vf, tyy)), qy), sy));
    }
#pragma unroll
    for (int k = 0; k < NV; ++k) {
        const double wl = w[ws(b, n, k, jL, iL)], wr = w[ws(b, n, k, jR, iR)];
        const double wll = w[ws(b, n, k, jL - dj, iL - di)], wrr = w[ws(b, n, k, jR + dj, iR + di)];
        const double fc = mul(0.5, add(FL[k], FR[k]));
        const double d = sub(mul(eps2, sub(wr, wl)), mul(eps4, sub(add(sub(wrr, mul(3.0, wr)), mul(3.0, wl)), wll)));
        out[k] = visc ? sub(sub(fc, d), fv[k]) : sub(fc, d);
    }
}

__global__ void ns_residual_kernel(hbns_args a, const double *w) {
    // grid.y = block, grid.z = snapshot; x over interior cells (i fastest)
    const hbns_block &b = a.blocks[blockIdx.y];
    const int n = blockIdx.z;
    const int g = a.Pg > 1 ? n : 0;
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= b.ni * b.nj) return;
    const int i = t % b.ni + 1, j = t / b.ni + 1;
    const double *gi = a.moving ? a.gi : nullptr;
    const double *gj = a.moving ? a.gj : nullptr;
    double fe[NV], fw[NV], fn[NV], fs[NV];
    face_flux(a, b, w, n, g, j, i, 0, 1, a.six[fi(b, g, j, i)], a.siy[fi(b, g, j, i)], gi ? gi[fi(b, g, j, i)] : 0.0,
              fe);
    face_flux(a, b, w, n, g, j, i - 1, 0, 1, a.six[fi(b, g, j, i - 1)], a.siy[fi(b, g, j, i - 1)],
              gi ? gi[fi(b, g, j, i - 1)] : 0.0, fw);
    face_flux(a, b, w, n, g, j, i, 1, 0, a.sjx[fj(b, g, j, i)], a.sjy[fj(b, g, j, i)], gj ? gj[fj(b, g, j, i)] : 0.0,
              fn);
    face_flux(a, b, w, n, g, j - 1, i, 1, 0, a.sjx[fj(b, g, j - 1, i)], a.sjy[fj(b, g, j - 1, i)],
              gj ? gj[fj(b, g, j - 1, i)] : 0.0, fs);
#pragma unroll
    for (int k = 0; k < NV; ++k) a.r[rs(b, n, k, j, i)] = sub(add(sub(fe[k], fw[k]), fn[k]), fs[k]);
}

__global__ void ns_timestep_kernel(hbns_args a, const double *w) {
    const hbns_block &b = a.blocks[blockIdx.y];
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= b.ni * b.nj) return;
    const int i = t % b.ni + 1, j = t / b.ni + 1;
    const int64_t st = (int64_t)(b.nj + 4) * (b.ni + 4);
    const bool mv = a.moving != 0;
    double best = 0.0;
    for (int n = 0; n < a.P; ++n) {
        const int g = a.Pg > 1 ? n : 0;
        const Prim q = prim(w + ws(b, n, 0, j, i), st);
        const double ax = a.six[fi(b, g, j, i - 1)], ay = a.siy[fi(b, g, j, i - 1)];
        const double bx = a.six[fi(b, g, j, i)], by = a.siy[fi(b, g, j, i)];
        const double cx = a.sjx[fj(b, g, j - 1, i)], cy = a.sjy[fj(b, g, j - 1, i)];
        const double dx = a.sjx[fj(b, g, j, i)], dy = a.sjy[fj(b, g, j, i)];
        const double ga = mv ? a.gi[fi(b, g, j, i - 1)] : 0.0, gb = mv ? a.gi[fi(b, g, j, i)] : 0.0;
        const double gc = mv ? a.gj[fj(b, g, j - 1, i)] : 0.0, gd = mv ? a.gj[fj(b, g, j, i)] : 0.0;
        const double la = add(fabs(sub(add(mul(q.u, ax), mul(q.v, ay)), ga)), mul(q.c, __dsqrt_rn(add(mul(ax, ax), mul(ay, ay)))));
        const double lb = add(fabs(sub(add(mul(q.u, bx), mul(q.v, by)), gb)), mul(q.c, __dsqrt_rn(add(mul(bx, bx), mul(by, by)))));
        const double lc = add(fabs(sub(add(mul(q.u, cx), mul(q.v, cy)), gc)), mul(q.c, __dsqrt_rn(add(mul(cx, cx), mul(cy, cy)))));
        const double ld = add(fabs(sub(add(mul(q.u, dx), mul(q.v, dy)), gd)), mul(q.c, __dsqrt_rn(add(mul(dx, dx), mul(dy, dy)))));
        const double V = a.vol[cc(b, g, j, i)];
        double den = add(mul(0.5, add(la, lb)), mul(0.5, add(lc, ld)));
        if (a.mu > 0.0) {
            const double sxi = mul(0.5, add(ax, bx)), syi = mul(0.5, add(ay, by));
            const double sxj = mul(0.5, add(cx, dx)), syj = mul(0.5, add(cy, dy));
            const double lv = mul(dv(mul(mul(2.0, GAMMA), a.mu), mul(PR, q.r)),
                                  dv(add(add(mul(sxi, sxi), mul(syi, syi)), add(mul(sxj, sxj), mul(syj, syj))), V));
            den = add(den, lv);
        }
        den = add(den, mul(a.omega_nh, V));
        const double tn = dv(mul(a.cfl, V), den);
        best = n == 0 ? tn : fmin(best, tn);
    }
    a.dt[b.dt_off + (int64_t)(j - 1) * b.ni + (i - 1)] = best;
}

constexpr int UPD_THREADS = 256;

// one thread per (cell, variable k), all P snapshots: each W_m is loaded once
// for the P outputs of the HB source
template <int P>
__global__ void __launch_bounds__(UPD_THREADS) ns_update_kernel(hbns_args a, const double *w_in, const double *w0,
                                                                  double *w_out, double coef, int want_norm) {
    // grid.y = block, grid.z = variable; x over interior cells
    __shared__ double red[UPD_THREADS];
    const hbns_block &b = a.blocks[blockIdx.y];
    const int k = blockIdx.z;
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    double sq = 0.0;
    if (t < b.ni * b.nj) {
        const int i = t % b.ni + 1, j = t / b.ni + 1;
        double wm[P];
#pragma unroll
        for (int m = 0; m < P; ++m) wm[m] = w_in[ws(b, m, k, j, i)];
        const double dtc = a.dt[b.dt_off + (int64_t)(j - 1) * b.ni + (i - 1)];
#pragma unroll
        for (int n = 0; n < P; ++n) {
            const int g = a.Pg > 1 ? n : 0;
            const double V = a.vol[cc(b, g, j, i)];
            double s = mul(a.dmat[n * P], wm[0]);
#pragma unroll
            for (int m = 1; m < P; ++m) s = add(s, mul(a.dmat[n * P + m], wm[m]));
            const double R = add(a.r[rs(b, n, k, j, i)], mul(V, s));
            if (want_norm && k == 0) sq = __fma_rn(R, R, sq);
            const double v = sub(w0[ws(b, n, k, j, i)], mul(dv(mul(coef, dtc), V), R));
            w_out[ws(b, n, k, j, i)] = v;
            if (!isfinite(v)) {
                const long long lin = (((long long)(n * NV + k) * b.nj + (j - 1)) * b.ni) + (i - 1);
                atomicMin(a.status + blockIdx.y, (unsigned long long)lin);
            }
        }
    }
    if (want_norm && k == 0) {
        red[threadIdx.x] = sq;
        __syncthreads();
        for (int s2 = UPD_THREADS / 2; s2 > 0; s2 >>= 1) {
            if (threadIdx.x < s2) red[threadIdx.x] = add(red[threadIdx.x], red[threadIdx.x + s2]);
            __syncthreads();
        }
        if (threadIdx.x == 0) a.norm_part[b.part_off + blockIdx.x] = red[0];
    }
}

// stage-1 norm: one warp per block folds that block's CTA partials in a fixed
// lane-strided order and shuffle tree; one thread then folds blocks in order
__global__ void ns_norm_kernel(hbns_args a, int iter, int ctas) {
    __shared__ double blk_sum[1024];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    for (int bk = warp; bk < a.nblocks; bk += nw) {
        const hbns_block &b = a.blocks[bk];
        const int used = (int)(((int64_t)b.ni * b.nj + UPD_THREADS - 1) / UPD_THREADS);
        double s = 0.0;
        for (int c = lane; c < used && c < ctas; c += 32) s = add(s, a.norm_part[b.part_off + c]);
        for (int o = 16; o > 0; o >>= 1) s = add(s, __shfl_down_sync(0xffffffffu, s, o));
        if (lane == 0) blk_sum[bk] = s;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int bk = 0; bk < a.nblocks; ++bk) s = add(s, blk_sum[bk]);
        a.norms[iter] = __dsqrt_rn(s);
    }
}

__global__ void ns_forces_kernel(hbns_args a, const double *w, int iter) {
    const int n = threadIdx.x;
    if (n >= a.P) return;
    const int g = a.Pg > 1 ? n : 0;
    double fx = 0.0, fy = 0.0;
    for (int bk = 0; bk < a.nblocks; ++bk) {
        const hbns_block &b = a.blocks[bk];
        const int64_t st = (int64_t)(b.nj + 4) * (b.ni + 4);
        for (int side = 0; side < 4; ++side) {
            if (b.kinds[side] != HBNS_NOSLIP && b.kinds[side] != HBNS_SLIP) continue;
            const int len = side < 2 ? b.ni : b.nj;
            for (int e = 1; e <= len; ++e) {
                int ci, cj;
                double sx, sy;
                if (side == 0) { ci = e; cj = 1; sx = a.sjx[fj(b, g, 0, e)]; sy = a.sjy[fj(b, g, 0, e)]; }
                else if (side == 1) { ci = e; cj = b.nj; sx = a.sjx[fj(b, g, b.nj, e)]; sy = a.sjy[fj(b, g, b.nj, e)]; }
                else if (side == 2) { ci = 1; cj = e; sx = a.six[fi(b, g, e, 0)]; sy = a.siy[fi(b, g, e, 0)]; }
                else { ci = b.ni; cj = e; sx = a.six[fi(b, g, e, b.ni)]; sy = a.siy[fi(b, g, e, b.ni)]; }
                const Prim q = prim(w + ws(b, n, 0, cj, ci), st);
                fx = add(fx, mul(q.p, sx));
                fy = add(fy, mul(q.p, sy));
            }
        }
    }
    a.forces[((int64_t)iter * a.P + n) * 2] = fx;
    a.forces[((int64_t)iter * a.P + n) * 2 + 1] = fy;
}

int check(const char *what) { return hbgpu_check_launch(what); }

}  // namespace hbns

using namespace hbns;

extern "C" int hbns_boundaries(const hbns_args *a, int32_t slot, void *stream) {
    if (a == nullptr || slot < 0 || slot > 2) {
        hbgpu_set_error("hbns_boundaries: bad arguments");
        return HBGPU_ERR_ARG;
    }
    cudaStream_t s = (cudaStream_t)stream;
    const int maxlen = a->max_len;
    ns_bc_kernel<<<dim3((8 * maxlen + 127) / 128, a->nblocks, a->P), 128, 0, s>>>(*a, a->w[slot]);
    ns_corner_kernel<<<dim3(1, a->nblocks, a->P * NV), 32, 0, s>>>(*a, a->w[slot]);
    hbgpu_count_launch(2);
    return check("hbns_boundaries");
}

extern "C" int hbns_timestep(const hbns_args *a, int32_t slot, void *stream) {
    ns_timestep_kernel<<<dim3((a->max_cells + 127) / 128, a->nblocks), 128, 0, (cudaStream_t)stream>>>(*a, a->w[slot]);
    hbgpu_count_launch(1);
    return check("hbns_timestep");
}

extern "C" int hbns_residual(const hbns_args *a, int32_t slot, void *stream) {
    cudaStream_t s = (cudaStream_t)stream;
    const int halo_cells = (a->max_len + 4) * (a->max_len + 4);
    ns_prim_kernel<<<dim3((halo_cells + 127) / 128, a->nblocks, a->P), 128, 0, s>>>(*a, a->w[slot]);
    ns_residual_kernel<<<dim3((a->max_cells + 127) / 128, a->nblocks, a->P), 128, 0, s>>>(*a, a->w[slot]);
    hbgpu_count_launch(2);
    return check("hbns_residual");
}

extern "C" int hbns_update(const hbns_args *a, int32_t slot_in, int32_t slot_out, double coef, int32_t iter,
                           int32_t want_norm, void *stream) {
    cudaStream_t s = (cudaStream_t)stream;
    const int ctas = (a->max_cells + UPD_THREADS - 1) / UPD_THREADS;
    if (a->nblocks > 1024) {
        hbgpu_set_error("hbns_update: at most 1024 blocks");
        return HBGPU_ERR_ARG;
    }
    const dim3 grid(ctas, a->nblocks, NV);
    switch (a->P) {
        case 1: ns_update_kernel<1><<<grid, UPD_THREADS, 0, s>>>(*a, a->w[slot_in], a->w[0], a->w[slot_out], coef, want_norm); break;
        case 3: ns_update_kernel<3><<<grid, UPD_THREADS, 0, s>>>(*a, a->w[slot_in], a->w[0], a->w[slot_out], coef, want_norm); break;
        case 5: ns_update_kernel<5><<<grid, UPD_THREADS, 0, s>>>(*a, a->w[slot_in], a->w[0], a->w[slot_out], coef, want_norm); break;
        case 7: ns_update_kernel<7><<<grid, UPD_THREADS, 0, s>>>(*a, a->w[slot_in], a->w[0], a->w[slot_out], coef, want_norm); break;
        case 9: ns_update_kernel<9><<<grid, UPD_THREADS, 0, s>>>(*a, a->w[slot_in], a->w[0], a->w[slot_out], coef, want_norm); break;
        default:
            hbgpu_set_error("hbns_update: P = %d not templated (1..9 odd)", a->P);
            return HBGPU_ERR_UNSUPPORTED;
    }
    int n = 1;
    if (want_norm) {
        ns_norm_kernel<<<1, 1024, 0, s>>>(*a, iter, ctas);
        ++n;
    }
    hbgpu_count_launch(n);
    return check("hbns_update");
}

extern "C" int hbns_forces(const hbns_args *a, int32_t iter, void *stream) {
    ns_forces_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(*a, a->w[0], iter);
    hbgpu_count_launch(1);
    return check("hbns_forces");
}
