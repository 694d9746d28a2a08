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
//   ns_flux_kernel      R of a TJ x TI tile and one snapshot per CTA: the
//                       state with its 2-cell ring staged in shared memory,
//                       primitives once per staged cell, sensors once per
//                       (cell, direction), every face flux once
//   ns_update_kernel    HB source + RK update, one thread per (cell,
//                       variable) for all snapshots; stage-1 R_rho^2 partials
//                       per CTA, folded by ns_norm_kernel (a warp per block)
//   ns_forces_kernel    wall pressure forces, one thread per snapshot
// Cut halos move with hbgpu_halo (two directions per cut and layer).

#include "hb_tma.cuh"

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

// ---- residual: one CTA per (tile of TJ x TI cells, snapshot) ---------------------------
//
// The tile's state with its two-cell halo ring is staged in shared memory;
// primitives are formed once per staged cell, the JST pressure sensor once per
// (cell, direction), and every face flux once -- the two cells beside a face
// read the same value (the thread-per-cell form computed each face twice and
// each sensor up to four times).  Geometry comes through L1/L2: the face
// normals are read once per face, the cell centres of the viscous diamond
// from L1.  The per-point arithmetic is the specification's, operation for
// operation, so R is bitwise the thread-per-cell kernel's (and the oracle's).

constexpr int TI = 32, TJ = 8;               // tile columns, rows
constexpr int RW = TI + 4, RH = TJ + 4;      // staged region with the 2-cell ring
constexpr int FLUX_THREADS = 288;            // 9 warps: 264 i-faces / 288 j-faces per pass

struct FluxSmem {
    double w[NV][RH][RW];          // conservative state
    double pr[5][RH][RW];          // u, v, p, c, e
    double xc[RH - 2][RW - 2];     // cell centres of the 1-cell ring region (viscous)
    double yc[RH - 2][RW - 2];
    double nxi[TJ][TI + 1], nyi[TJ][TI + 1], gfi[TJ][TI + 1];   // i-face normals, grid flux
    double nxj[TJ + 1][TI], nyj[TJ + 1][TI], gfj[TJ + 1][TI];   // j-face normals, grid flux
    double nui[TJ][TI + 2];        // sensor along i: tile rows, columns i0-1 .. i0+TI
    double nuj[TJ + 2][TI];        // sensor along j: rows j0-1 .. j0+TJ, tile columns
    double fi[NV][TJ][TI + 1];     // i-face fluxes: face k between cells i0-1+k and i0+k
    double fj[NV][TJ + 1][TI];     // j-face fluxes: face k between rows j0-1+k and j0+k
};

// one 8-byte global -> shared copy, asynchronous (LDGSTS): a CTA issues all
// of its staging copies before waiting once
__device__ __forceinline__ void cp8(double *sdst, const double *gsrc) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(sdst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

__device__ __forceinline__ double sensor(double pm, double pc, double pp) {
    // nu_X = |(p_{X+1} - 2 p_X) + p_{X-1}| / ((p_{X+1} + 2 p_X) + p_{X-1})
    return dv(fabs(add(sub(pp, mul(2.0, pc)), pm)), add(add(pp, mul(2.0, pc)), pm));
}

// flux through the face between region cells L = (ry, rx) and R = L + (dj, di)
template <bool VISC>
__device__ __forceinline__ void tile_face(const hbns_args &a, const FluxSmem &S, int ry, int rx, int dj, int di,
                                          double sx, double sy, double gf, double nuL, double nuR, double *out) {
    const int ryR = ry + dj, rxR = rx + di;
    const double Lr = S.w[0][ry][rx], Lru = S.w[1][ry][rx], Lrv = S.w[2][ry][rx], Lre = S.w[3][ry][rx];
    const double Rr = S.w[0][ryR][rxR], Rru = S.w[1][ryR][rxR], Rrv = S.w[2][ryR][rxR], Rre = S.w[3][ryR][rxR];
    const double Lu = S.pr[0][ry][rx], Lv = S.pr[1][ry][rx], Lp = S.pr[2][ry][rx], Lc = S.pr[3][ry][rx];
    const double Ru = S.pr[0][ryR][rxR], Rv = S.pr[1][ryR][rxR], Rp = S.pr[2][ryR][rxR], Rc = S.pr[3][ryR][rxR];
    const double unL = add(mul(Lu, sx), mul(Lv, sy)), unR = add(mul(Ru, sx), mul(Rv, sy));
    const double urL = sub(unL, gf), urR = sub(unR, gf);
    const double FL[NV] = {mul(Lr, urL), add(mul(Lru, urL), mul(Lp, sx)), add(mul(Lrv, urL), mul(Lp, sy)),
                           add(mul(Lre, urL), mul(Lp, unL))};
    const double FR[NV] = {mul(Rr, urR), add(mul(Rru, urR), mul(Rp, sx)), add(mul(Rrv, urR), mul(Rp, sy)),
                           add(mul(Rre, urR), mul(Rp, unR))};
    const double sa = __dsqrt_rn(add(mul(sx, sx), mul(sy, sy)));
    const double lamL = add(fabs(urL), mul(Lc, sa)), lamR = add(fabs(urR), mul(Rc, sa));
    const double lam = mul(0.5, add(lamL, lamR));
    const double eps2 = mul(mul(K2, lam), fmax(nuL, nuR));
    const double eps4 = fmax(0.0, sub(mul(K4, lam), eps2));
    double fv[NV] = {0.0, 0.0, 0.0, 0.0};
    if (VISC) {
        const int tj = di, ti = dj;   // i-face: rows +-1; j-face: columns +-1
        // centres: ring-1 region coordinates are the region's minus one
        const int cy = ry - 1, cx = rx - 1, cyR = ryR - 1, cxR = rxR - 1;
        const double xL = S.xc[cy][cx], xR = S.xc[cyR][cxR];
        const double yL = S.yc[cy][cx], yR = S.yc[cyR][cxR];
        const double xLp = S.xc[cy + tj][cx + ti], xRp = S.xc[cyR + tj][cxR + ti];
        const double xLm = S.xc[cy - tj][cx - ti], xRm = S.xc[cyR - tj][cxR - ti];
        const double yLp = S.yc[cy + tj][cx + ti], yRp = S.yc[cyR + tj][cxR + ti];
        const double yLm = S.yc[cy - tj][cx - ti], yRm = S.yc[cyR - tj][cxR - ti];
        const double x_a = sub(xR, xL), y_a = sub(yR, yL);
        const double x_b = mul(0.25, sub(add(xLp, xRp), add(xLm, xRm)));
        const double y_b = mul(0.25, sub(add(yLp, yRp), add(yLm, yRm)));
        const double jac = sub(mul(x_a, y_b), mul(x_b, y_a));
        // u, v, e of the four diamond cells beside L and R
        const int pLy = ry + tj, pLx = rx + ti, mLy = ry - tj, mLx = rx - ti;
        const int pRy = ryR + tj, pRx = rxR + ti, mRy = ryR - tj, mRx = rxR - ti;
        const double ua = sub(Ru, Lu);
        const double ub = mul(0.25, sub(add(S.pr[0][pLy][pLx], S.pr[0][pRy][pRx]), add(S.pr[0][mLy][mLx], S.pr[0][mRy][mRx])));
        const double va = sub(Rv, Lv);
        const double vb = mul(0.25, sub(add(S.pr[1][pLy][pLx], S.pr[1][pRy][pRx]), add(S.pr[1][mLy][mLx], S.pr[1][mRy][mRx])));
        const double ea = sub(S.pr[4][ryR][rxR], S.pr[4][ry][rx]);
        const double eb = mul(0.25, sub(add(S.pr[4][pLy][pLx], S.pr[4][pRy][pRx]), add(S.pr[4][mLy][mLx], S.pr[4][mRy][mRx])));
        const double ux = dv(sub(mul(ua, y_b), mul(ub, y_a)), jac), uy = dv(sub(mul(ub, x_a), mul(ua, x_b)), jac);
        const double vx = dv(sub(mul(va, y_b), mul(vb, y_a)), jac), vy = dv(sub(mul(vb, x_a), mul(va, x_b)), jac);
        const double ex = dv(sub(mul(ea, y_b), mul(eb, y_a)), jac), ey = dv(sub(mul(eb, x_a), mul(ea, x_b)), jac);
        const double mu = a.mu;
        const double div = add(ux, vy);
        const double t23 = 2.0 / 3.0;
        const double txx = mul(mu, sub(mul(2.0, ux), mul(t23, div)));
        const double tyy = mul(mu, sub(mul(2.0, vy), mul(t23, div)));
        const double txy = mul(mu, add(uy, vx));
        const double kq = a.kq;   // (mu * gamma) / Pr, formed once on the host
        const double qx = -mul(kq, ex), qy = -mul(kq, ey);
        const double uf = mul(0.5, add(Lu, Ru)), vf = mul(0.5, add(Lv, Rv));
        fv[1] = add(mul(txx, sx), mul(txy, sy));
        fv[2] = add(mul(txy, sx), mul(tyy, sy));
        fv[3] = add(mul(sub(add(mul(uf, txx), mul(vf, txy)), qx), sx), mul(sub(add(mul(uf, txy), mul(vf, tyy)), qy), sy));
    }
#pragma unroll
    for (int k = 0; k < NV; ++k) {
        const double wl = S.w[k][ry][rx], wr = S.w[k][ryR][rxR];
        const double wll = S.w[k][ry - dj][rx - di], wrr = S.w[k][ryR + dj][rxR + di];
        const double fc = mul(0.5, add(FL[k], FR[k]));
        const double d = sub(mul(eps2, sub(wr, wl)), mul(eps4, sub(add(sub(wrr, mul(3.0, wr)), mul(3.0, wl)), wll)));
        out[k] = VISC ? sub(sub(fc, d), fv[k]) : sub(fc, d);
    }
}

// one row of `count` (<= 64) staged values, lane-strided; columns past
// `last` read column `last` (clamped to the block's array)
__device__ __forceinline__ void stage_row(double *sdst, const double *grow, int count, int last, int lane) {
    cp8(sdst + lane, grow + min(lane, last));
    if (lane + 32 < count) cp8(sdst + lane + 32, grow + min(lane + 32, last));
}

// Thread mapping: lane = tile column, warp = row (TI = 32 = warp width), so
// staging, primitives, sensors and faces need no index division; the 9th
// warp takes the 8 east-most i-faces and the last j-face row.
// CTAs per SM the register budget is sized for: 3 of 9 warps (the register
// file is split over the 4 schedulers, so <= 72 registers; a few spill, and
// the extra warps still win: C4 231 -> 223, C3 15.6 -> 15.2 ms/iteration
// against 2).  HBNS_FLUX_MINB overrides it in measurement builds.
#ifndef HBNS_FLUX_MINB
#define HBNS_FLUX_MINB 3
#endif

template <bool VISC>
__global__ void __launch_bounds__(FLUX_THREADS, HBNS_FLUX_MINB) ns_flux_kernel(hbns_args a, const double *w) {
    // grid.x = tile * P + snapshot (snapshots of a tile adjacent: the same
    // geometry when the mesh is fixed), grid.y = block
    extern __shared__ __align__(16) unsigned char smem_raw[];
    FluxSmem &S = *reinterpret_cast<FluxSmem *>(smem_raw);
    const hbns_block b = a.blocks[blockIdx.y];
    const int n = blockIdx.x % a.P;
    const int tile = blockIdx.x / a.P;
    const int tiles_i = (b.ni + TI - 1) / TI;
    if (tile >= tiles_i * ((b.nj + TJ - 1) / TJ)) return;
    const int i0 = (tile % tiles_i) * TI + 1, j0 = (tile / tiles_i) * TJ + 1;
    const int g = a.Pg > 1 ? n : 0;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr int NW = FLUX_THREADS / 32;
    // 1. stage, all copies in flight at once: the state of region cells
    //    (j0-2 .. j0+TJ+1) x (i0-2 .. i0+TI+1), clamped to the block's array
    //    (the clamped cells feed no face); the tile's face normals and grid
    //    fluxes; the cell centres of the 1-cell ring (viscous)
    {
        const int ilast = b.ni + 2 - (i0 - 2);   // region column of array column ni+2
        for (int row = warp; row < NV * RH; row += NW) {
            const int k = row / RH, r = row - k * RH;
            stage_row(S.w[k][r], w + ws(b, n, k, min(j0 - 2 + r, b.nj + 2), i0 - 2), RW, ilast, lane);
        }
        const int flast = b.ni - (i0 - 1);       // i-face column of face ni
        for (int r = warp; r < TJ; r += NW) {
            const int64_t f = fi(b, g, min(j0 + r, b.nj), i0 - 1);
            stage_row(S.nxi[r], a.six + f, TI + 1, flast, lane);
            stage_row(S.nyi[r], a.siy + f, TI + 1, flast, lane);
            if (a.moving) stage_row(S.gfi[r], a.gi + f, TI + 1, flast, lane);
        }
        const int jlast = b.ni - i0;             // j-face / tile column of cell ni
        for (int r = warp; r <= TJ; r += NW) {
            const int64_t f = fj(b, g, min(j0 - 1 + r, b.nj), i0);
            stage_row(S.nxj[r], a.sjx + f, TI, jlast, lane);
            stage_row(S.nyj[r], a.sjy + f, TI, jlast, lane);
            if (a.moving) stage_row(S.gfj[r], a.gj + f, TI, jlast, lane);
        }
        if (VISC) {
            const int clast = b.ni + 1 - (i0 - 1);
            for (int r = warp; r < RH - 2; r += NW) {
                const int64_t o = cc(b, g, min(j0 - 1 + r, b.nj + 1), i0 - 1);
                stage_row(S.xc[r], a.xc + o, RW - 2, clast, lane);
                stage_row(S.yc[r], a.yc + o, RW - 2, clast, lane);
            }
        }
    }
    cp_wait_all();
    __syncthreads();
    // 2. primitives of every staged cell (nsflow: u, v, p, c, e)
    for (int t = threadIdx.x; t < RH * RW; t += FLUX_THREADS) {
        const int r = t / RW, c = t - r * RW;
        const double q_r = S.w[0][r][c], q_ru = S.w[1][r][c], q_rv = S.w[2][r][c], q_re = S.w[3][r][c];
        const double u = dv(q_ru, q_r), v = dv(q_rv, q_r);
        const double p = mul(GAMMA - 1.0, sub(q_re, mul(0.5, add(mul(q_ru, u), mul(q_rv, v)))));
        S.pr[0][r][c] = u;
        S.pr[1][r][c] = v;
        S.pr[2][r][c] = p;
        S.pr[3][r][c] = __dsqrt_rn(dv(mul(GAMMA, p), q_r));
        S.pr[4][r][c] = dv(p, mul(GAMMA - 1.0, q_r));
    }
    __syncthreads();
    // 3. JST sensors of the cells beside the tile's faces
    constexpr int NSI = TJ * (TI + 2), NSJ = (TJ + 2) * TI;
    for (int t = threadIdx.x; t < NSI + NSJ; t += FLUX_THREADS) {
        if (t < NSI) {
            const int r = t / (TI + 2), c = t - r * (TI + 2);   // cell (j0 + r, i0 - 1 + c)
            S.nui[r][c] = sensor(S.pr[2][r + 2][c], S.pr[2][r + 2][c + 1], S.pr[2][r + 2][c + 2]);
        } else {
            const int u = t - NSI, r = u / TI, c = u % TI;      // cell (j0 - 1 + r, i0 + c)
            S.nuj[r][c] = sensor(S.pr[2][r][c + 2], S.pr[2][r + 1][c + 2], S.pr[2][r + 2][c + 2]);
        }
    }
    __syncthreads();
    // 4. face fluxes, one i-face and one j-face per thread, both evaluated
    //    unconditionally (indices clamped into the staged region) so that the
    //    two dependency chains interleave; only real faces are stored.
    //    Warp w < TJ: i-faces of row w (faces 0..31); warp TJ: face 32 of
    //    every row (lanes 0..TJ-1).  Every warp w: j-face row w.
    {
        const bool mv = a.moving != 0;
        const int ri = warp < TJ ? warp : min(lane, TJ - 1), ci = warp < TJ ? lane : TI;
        const bool live_i = (warp < TJ || lane < TJ) && j0 + ri <= b.nj && i0 - 1 + ci <= b.ni;
        const int rj = warp, cj = lane;
        const bool live_j = j0 - 1 + rj <= b.nj && i0 + cj <= b.ni;
        double oi[NV], oj[NV];
        tile_face<VISC>(a, S, ri + 2, ci + 1, 0, 1, S.nxi[ri][ci], S.nyi[ri][ci], mv ? S.gfi[ri][ci] : 0.0,
                        S.nui[ri][ci], S.nui[ri][ci + 1], oi);
        tile_face<VISC>(a, S, rj + 1, cj + 2, 1, 0, S.nxj[rj][cj], S.nyj[rj][cj], mv ? S.gfj[rj][cj] : 0.0,
                        S.nuj[rj][cj], S.nuj[rj + 1][cj], oj);
        if (live_i) {
#pragma unroll
            for (int k = 0; k < NV; ++k) S.fi[k][ri][ci] = oi[k];
        }
        if (live_j) {
#pragma unroll
            for (int k = 0; k < NV; ++k) S.fj[k][rj][cj] = oj[k];
        }
    }
    __syncthreads();
    // 5. R = ((F_{i+1/2} - F_{i-1/2}) + F_{j+1/2}) - F_{j-1/2}
    if (warp < TJ) {
        const int r = warp, c = lane;
        const int j = j0 + r, i = i0 + c;
        if (j <= b.nj && i <= b.ni) {
#pragma unroll
            for (int k = 0; k < NV; ++k)
                a.r[rs(b, n, k, j, i)] = sub(add(sub(S.fi[k][r][c + 1], S.fi[k][r][c]), S.fj[k][r + 1][c]), S.fj[k][r][c]);
        }
    }
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

// wall pressure forces: one CTA per snapshot.  The wall faces in the
// specification's order (blocks ascending, sides south/north/west/east, face
// cells ascending) are taken in chunks: every thread forms p*Sx and p*Sy of
// its faces (each product rounded once), then thread 0 adds them in order --
// the fold is the only serial part.
constexpr int FORCE_THREADS = 256;
constexpr int FORCE_CHUNK = 1024;
constexpr int MAX_WALL_SEGS = 4 * 256;

__global__ void __launch_bounds__(FORCE_THREADS) ns_forces_kernel(hbns_args a, const double *w, int iter) {
    __shared__ double px[FORCE_CHUNK], py[FORCE_CHUNK];
    __shared__ int seg_bs[MAX_WALL_SEGS], seg_end[MAX_WALL_SEGS];   // block * 4 + side, running end
    __shared__ int nseg_s;
    const int n = blockIdx.x;
    const int g = a.Pg > 1 ? n : 0;
    if (threadIdx.x == 0) {
        int ns = 0, end = 0;
        for (int bk = 0; bk < a.nblocks && ns < MAX_WALL_SEGS; ++bk) {
            const hbns_block &b = a.blocks[bk];
            for (int side = 0; side < 4; ++side) {
                if (b.kinds[side] != HBNS_NOSLIP && b.kinds[side] != HBNS_SLIP) continue;
                end += side < 2 ? b.ni : b.nj;
                seg_bs[ns] = bk * 4 + side;
                seg_end[ns] = end;
                ++ns;
            }
        }
        nseg_s = ns;
    }
    __syncthreads();
    const int nseg = nseg_s;
    const int total = nseg > 0 ? seg_end[nseg - 1] : 0;
    double fx = 0.0, fy = 0.0;
    for (int c0 = 0; c0 < total; c0 += FORCE_CHUNK) {
        int sg = 0;
        for (int t = c0 + threadIdx.x; t < min(total, c0 + FORCE_CHUNK); t += FORCE_THREADS) {
            while (t >= seg_end[sg]) ++sg;
            const int bk = seg_bs[sg] >> 2, side = seg_bs[sg] & 3;
            const hbns_block &b = a.blocks[bk];
            const int e = t - (sg > 0 ? seg_end[sg - 1] : 0) + 1;
            int ci, cj;
            double sx, sy;
            if (side == 0) { ci = e; cj = 1; sx = a.sjx[fj(b, g, 0, e)]; sy = a.sjy[fj(b, g, 0, e)]; }
            else if (side == 1) { ci = e; cj = b.nj; sx = a.sjx[fj(b, g, b.nj, e)]; sy = a.sjy[fj(b, g, b.nj, e)]; }
            else if (side == 2) { ci = 1; cj = e; sx = a.six[fi(b, g, e, 0)]; sy = a.siy[fi(b, g, e, 0)]; }
            else { ci = b.ni; cj = e; sx = a.six[fi(b, g, e, b.ni)]; sy = a.siy[fi(b, g, e, b.ni)]; }
            const Prim q = prim(w + ws(b, n, 0, cj, ci), (int64_t)(b.nj + 4) * (b.ni + 4));
            px[t - c0] = mul(q.p, sx);
            py[t - c0] = mul(q.p, sy);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            const int m = min(FORCE_CHUNK, total - c0);
            for (int e = 0; e < m; ++e) {
                fx = add(fx, px[e]);
                fy = add(fy, py[e]);
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        a.forces[((int64_t)iter * a.P + n) * 2] = fx;
        a.forces[((int64_t)iter * a.P + n) * 2 + 1] = fy;
    }
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
    if (a == nullptr || slot < 0 || slot > 2 || a->max_ni < 1 || a->max_nj < 1) {
        hbgpu_set_error("hbns_residual: bad arguments");
        return HBGPU_ERR_ARG;
    }
    static bool ready[hbgpu::HB_MAX_DEVICES][2];
    const int dev = hbgpu::current_device();
    if (dev < 0) return HBGPU_ERR_CUDA;
    const bool visc = a->mu > 0.0;
    const size_t smem = sizeof(FluxSmem);
    if (!ready[dev][visc]) {
        cudaError_t e = visc ? cudaFuncSetAttribute(ns_flux_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)
                             : cudaFuncSetAttribute(ns_flux_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return check("hbns_residual (smem attribute)");
        ready[dev][visc] = true;
    }
    const int64_t tiles = (int64_t)((a->max_ni + TI - 1) / TI) * ((a->max_nj + TJ - 1) / TJ);
    if (tiles * a->P > INT32_MAX || a->nblocks > 65535) {
        hbgpu_set_error("hbns_residual: grid too large");
        return HBGPU_ERR_ARG;
    }
    const dim3 grid((unsigned)(tiles * a->P), a->nblocks);
    cudaStream_t s = (cudaStream_t)stream;
    if (visc) ns_flux_kernel<true><<<grid, FLUX_THREADS, smem, s>>>(*a, a->w[slot]);
    else ns_flux_kernel<false><<<grid, FLUX_THREADS, smem, s>>>(*a, a->w[slot]);
    hbgpu_count_launch(1);
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
    if (a->nblocks > 256) {
        hbgpu_set_error("hbns_forces: at most 256 blocks");
        return HBGPU_ERR_ARG;
    }
    ns_forces_kernel<<<a->P, FORCE_THREADS, 0, (cudaStream_t)stream>>>(*a, a->w[0], iter);
    hbgpu_count_launch(1);
    return check("hbns_forces");
}
