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
//   ns_stage_kernel     one RK stage of a TJ x TI tile, all snapshots, per
//                       CTA: per snapshot the state with its 2-cell ring
//                       staged in shared memory, primitives once per staged
//                       cell, sensors once per (cell, direction), every face
//                       flux once, R_n to an L2-resident scratch (stage 1:
//                       the local time step folded over the snapshots); then
//                       HB source + RK update of the tile and the stage-1
//                       norm partial (folded by ns_norm_kernel)
//   ns_norm_kernel      per block the tile partials (a warp), blocks in order
//   ns_forces_kernel    wall pressure forces, one CTA per snapshot
// Cut halos move with hbgpu_halo (two directions per cut and layer).

#include "hb_tma.cuh"

#include "hbns.h"

#include <type_traits>

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

constexpr int TI = HBNS_TILE_I, TJ = HBNS_TILE_J;   // tile columns, rows
constexpr int RW = TI + 4, RH = TJ + 4;      // staged region with the 2-cell ring
constexpr int FLUX_THREADS = 288;            // 9 warps: 264 i-faces / 288 j-faces per pass
static_assert(RW % 2 == 0, "16-byte staging chunks");

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
    double dmat[HBGPU_MAX_TEMPLATED_P * HBGPU_MAX_TEMPLATED_P];   // HB matrix D (stage kernel)
};

// one 8-byte global -> shared copy, asynchronous (LDGSTS): a CTA issues all
// of its staging copies before waiting once
__device__ __forceinline__ void cp8(double *sdst, const double *gsrc) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(sdst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gsrc) : "memory");
}
// 16-byte form (both addresses 16-byte aligned), past L1: staged values are read once per CTA
__device__ __forceinline__ void cp16(double *sdst, const double *gsrc) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(sdst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gsrc) : "memory");
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
// CTAs per SM the register budget is sized for (9 warps each; the register
// file is split over the 4 schedulers, so 3 CTAs mean <= 72 registers and 2
// <= 96).  Measured on the fused stage kernel: Euler 3 (C4 201 vs 210 ms per
// iteration with 2), viscous 2 (C3 13.9 vs 14.9, C1 0.44 vs 0.50 ms).
// HBNS_FLUX_MINB overrides both in measurement builds.
#ifndef HBNS_UPDATE_LAZY   // update-step load schedule (see the update step), Euler / viscous
#define HBNS_UPDATE_LAZY 2
#endif
#ifndef HBNS_UPDATE_LAZY_VISC
#define HBNS_UPDATE_LAZY_VISC 0
#endif

#ifndef HBNS_DISCARD   // measurement builds may keep the residual scratch's write-backs
#define HBNS_DISCARD 1
#endif

// The RK stage of one TJ x TI tile, all snapshots, in one CTA (grid.x =
// tile, grid.y = block).  Per snapshot n: stage W_n with its 2-cell ring
// (and, once per tile unless the mesh moves, the face normals and cell
// centres), form the face fluxes, write R_n = sum of face fluxes to the
// residual pool -- an L2-resident scratch: this CTA reads it back moments
// later -- and, in the first stage, fold the cell's local time step (the
// specification's dt, min over snapshots, from the iteration's start state
// that stage 1 reads).  Then the update of the tile, thread = cell, for
// every (variable, snapshot): the HB source V sum_m D[n][m] W_m (m
// ascending) added to R_n, W^(s) = W^0 - (alpha_s dt / V) R.  The time-step
// and update kernels of the unfused schedule are gone: their inputs are
// already on chip (primitives, normals) or in L2 (R, W_m).
template <bool VISC, int P, int MINB, bool DSHARE>
__global__ void __launch_bounds__(FLUX_THREADS, MINB)
    ns_stage_kernel(hbns_args a, const double *w, const double *w0, double *w_out, double coef, int first, int iter) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    FluxSmem &S = *reinterpret_cast<FluxSmem *>(smem_raw);
    __shared__ double red[FLUX_THREADS / 32];
    const hbns_block b = a.blocks[blockIdx.y];
    const int tile = blockIdx.x;
    const int tiles_i = (b.ni + TI - 1) / TI;
    if (tile >= tiles_i * ((b.nj + TJ - 1) / TJ)) return;
    const int i0 = (tile % tiles_i) * TI + 1, j0 = (tile / tiles_i) * TJ + 1;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr int NW = FLUX_THREADS / 32;
    const bool mv = a.moving != 0;
    // this thread's cell in the update and time-step steps (warps 0..TJ-1)
    const int cr = warp, cc_ = lane;
    const int cj = j0 + cr, ci = i0 + cc_;
    const bool cell_live = warp < TJ && cj <= b.nj && ci <= b.ni;
    double best = 0.0;   // stage 1: the cell's time step, min over snapshots
    const int gstage = (a.iter_dev ? *a.iter_dev : iter) * 4 + a.stage + 1;
    // Index arithmetic in 32 bits: offsets inside one snapshot of one block
    // (below 2^31 values: nsflow.NSRun refuses larger blocks) are ints; only the
    // per-snapshot base pointers are 64-bit, formed once per snapshot.
    const int wrow = b.ni + 4;                    // state / centre row pitch
    const int wplane = (b.nj + 4) * wrow;         // one (snapshot, variable) plane; one geometry snapshot of xc/yc/vol
    const int rplane = b.nj * b.ni;               // one residual plane
    const int cell_w = (cj + 1) * wrow + ci + 1;  // this thread's cell in a state plane (ws / cc)
    const int cell_r = (cj - 1) * b.ni + ci - 1;  // ... in a residual plane (rs)
    // 16-byte staging copies: even row pitch (every plane offset is then even,
    // i0 - 1 is a multiple of 32 and the pools are 256-byte aligned) and no
    // column clamp (the region ends inside the block's array)
    const bool wide = (b.ni & 1) == 0 && i0 + TI + 1 <= b.ni + 2 && ((uintptr_t)w & 15) == 0 && (b.w_off & 1) == 0;
    for (int t = threadIdx.x; t < P * P; t += FLUX_THREADS) S.dmat[t] = a.dmat[t];
    for (int n = 0; n < P; ++n) {
        const int g = a.Pg > 1 ? n : 0;
        const bool geo = n == 0 || a.Pg > 1;   // stage the geometry of snapshot g
        __syncthreads();                        // the previous snapshot's reads of S are done
        // 1. stage, all copies in flight at once: the state of region cells
        //    (j0-2 .. j0+TJ+1) x (i0-2 .. i0+TI+1), clamped to the block's
        //    array (the clamped cells feed no face); the tile's face normals
        //    and grid fluxes; the cell centres of the 1-cell ring (viscous)
        {
            const int ilast = b.ni + 2 - (i0 - 2);   // region column of array column ni+2
            const double *wn = w + b.w_off + (int64_t)n * NV * wplane + (i0 - 1);   // (n, 0, j = -1, i0 - 2)
            if (wide) {
                // the region's NV * RH rows of RW values as 16-byte chunks, lane-
                // contiguous over the whole CTA (864 chunks: 3 per thread);
                // S.w is dense, so chunk c lands at value 2 c
                constexpr int CPR = RW / 2;   // chunks per row
#pragma unroll
                for (int c = threadIdx.x; c < NV * RH * CPR; c += FLUX_THREADS) {
                    const int row = c / CPR, k = row / RH, r = row - k * RH;
                    cp16(&S.w[0][0][0] + 2 * c,
                         wn + k * wplane + min(j0 - 1 + r, b.nj + 3) * wrow + 2 * (c - row * CPR));
                }
            } else
#pragma unroll 1   // unrolled, the six row copies cost more (C4 185.8 vs 180.8 ms per iteration)
            for (int row = warp; row < NV * RH; row += NW) {
                const int k = row / RH, r = row - k * RH;
                stage_row(S.w[k][r], wn + k * wplane + min(j0 - 1 + r, b.nj + 3) * wrow, RW, ilast, lane);
            }
            if (geo) {
                const int flast = b.ni - (i0 - 1);       // i-face column of face ni
                for (int r = warp; r < TJ; r += NW) {
                    const int64_t f = fi(b, g, min(j0 + r, b.nj), i0 - 1);
                    stage_row(S.nxi[r], a.six + f, TI + 1, flast, lane);
                    stage_row(S.nyi[r], a.siy + f, TI + 1, flast, lane);
                    if (mv) stage_row(S.gfi[r], a.gi + f, TI + 1, flast, lane);
                }
                const int jlast = b.ni - i0;             // j-face / tile column of cell ni
                for (int r = warp; r <= TJ; r += NW) {
                    const int64_t f = fj(b, g, min(j0 - 1 + r, b.nj), i0);
                    stage_row(S.nxj[r], a.sjx + f, TI, jlast, lane);
                    stage_row(S.nyj[r], a.sjy + f, TI, jlast, lane);
                    if (mv) stage_row(S.gfj[r], a.gj + f, TI, jlast, lane);
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
            if (VISC) S.pr[4][r][c] = dv(p, mul(GAMMA - 1.0, q_r));   // e: the viscous heat flux only
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
        //    unconditionally (indices clamped into the staged region) so that
        //    the two dependency chains interleave; only real faces are stored.
        //    Warp w < TJ: i-faces of row w (faces 0..31); warp TJ: face 32 of
        //    every row (lanes 0..TJ-1).  Every warp w: j-face row w.
        {
            const int ri = warp < TJ ? warp : min(lane, TJ - 1), ci2 = warp < TJ ? lane : TI;
            const bool live_i = (warp < TJ || lane < TJ) && j0 + ri <= b.nj && i0 - 1 + ci2 <= b.ni;
            const int rj = warp, cj2 = lane;
            const bool live_j = j0 - 1 + rj <= b.nj && i0 + cj2 <= b.ni;
            double oi[NV], oj[NV];
            tile_face<VISC>(a, S, ri + 2, ci2 + 1, 0, 1, S.nxi[ri][ci2], S.nyi[ri][ci2], mv ? S.gfi[ri][ci2] : 0.0,
                            S.nui[ri][ci2], S.nui[ri][ci2 + 1], oi);
            tile_face<VISC>(a, S, rj + 1, cj2 + 2, 1, 0, S.nxj[rj][cj2], S.nyj[rj][cj2], mv ? S.gfj[rj][cj2] : 0.0,
                            S.nuj[rj][cj2], S.nuj[rj + 1][cj2], oj);
            if (live_i) {
#pragma unroll
                for (int k = 0; k < NV; ++k) S.fi[k][ri][ci2] = oi[k];
            }
            if (live_j) {
#pragma unroll
                for (int k = 0; k < NV; ++k) S.fj[k][rj][cj2] = oj[k];
            }
        }
        __syncthreads();
        // 5. R_n = ((F_{i+1/2} - F_{i-1/2}) + F_{j+1/2}) - F_{j-1/2}; stage 1:
        //    the local time step of snapshot n (nsflow: lambda_i, lambda_j,
        //    lambda_v, omega N_H V), folded into the min over snapshots
        if (cell_live) {
            const int r = cr, c = cc_;
            double *rn_ = a.r + b.r_off + (int64_t)n * NV * rplane + cell_r;
#pragma unroll
            for (int k = 0; k < NV; ++k)
                rn_[k * rplane] = sub(add(sub(S.fi[k][r][c + 1], S.fi[k][r][c]), S.fj[k][r + 1][c]), S.fj[k][r][c]);
            if (first) {
                const double qu = S.pr[0][r + 2][c + 2], qv = S.pr[1][r + 2][c + 2], qc = S.pr[3][r + 2][c + 2];
                const double ax = S.nxi[r][c], ay = S.nyi[r][c], bx = S.nxi[r][c + 1], by = S.nyi[r][c + 1];
                const double cx = S.nxj[r][c], cy = S.nyj[r][c], dx = S.nxj[r + 1][c], dy = S.nyj[r + 1][c];
                const double ga = mv ? S.gfi[r][c] : 0.0, gb = mv ? S.gfi[r][c + 1] : 0.0;
                const double gc = mv ? S.gfj[r][c] : 0.0, gd = mv ? S.gfj[r + 1][c] : 0.0;
                const double la = add(fabs(sub(add(mul(qu, ax), mul(qv, ay)), ga)), mul(qc, __dsqrt_rn(add(mul(ax, ax), mul(ay, ay)))));
                const double lb = add(fabs(sub(add(mul(qu, bx), mul(qv, by)), gb)), mul(qc, __dsqrt_rn(add(mul(bx, bx), mul(by, by)))));
                const double lc = add(fabs(sub(add(mul(qu, cx), mul(qv, cy)), gc)), mul(qc, __dsqrt_rn(add(mul(cx, cx), mul(cy, cy)))));
                const double ld = add(fabs(sub(add(mul(qu, dx), mul(qv, dy)), gd)), mul(qc, __dsqrt_rn(add(mul(dx, dx), mul(dy, dy)))));
                const double V = a.vol[b.c_off + (int64_t)g * wplane + cell_w];
                double den = add(mul(0.5, add(la, lb)), mul(0.5, add(lc, ld)));
                if (VISC) {
                    const double sxi = mul(0.5, add(ax, bx)), syi = mul(0.5, add(ay, by));
                    const double sxj = mul(0.5, add(cx, dx)), syj = mul(0.5, add(cy, dy));
                    const double lv = mul(dv(mul(mul(2.0, GAMMA), a.mu), mul(PR, S.w[0][r + 2][c + 2])),
                                          dv(add(add(mul(sxi, sxi), mul(syi, syi)), add(mul(sxj, sxj), mul(syj, syj))), V));
                    den = add(den, lv);
                }
                den = add(den, mul(a.omega_nh, V));
                const double tn = dv(mul(a.cfl, V), den);
                best = n == 0 ? tn : fmin(best, tn);
            }
        }
    }
    __syncthreads();   // R of every snapshot written (CTA-visible)
    // 6. HB source + RK update, thread = cell, for every (variable, snapshot).
    //    All of a variable's inputs are loaded before its first store (the
    //    output may be W^0 itself, stage 4), so the loads overlap.
    double sq = 0.0;
    if (cell_live) {
        const int64_t dti = b.dt_off + (int64_t)(cj - 1) * b.ni + (ci - 1);
        double dtc;
        if (first) {
            a.dt[dti] = best;
            dtc = best;
        } else {
            dtc = a.dt[dti];
        }
        // V and alpha_s dt / V: one value on a fixed mesh, per snapshot on a
        // moving one (recomputed per variable there: no register arrays)
        const double *volc = a.vol + b.c_off + cell_w;   // this cell, geometry snapshot 0
        const double V0 = volc[0];
        const double cdt0 = dv(mul(coef, dtc), V0);
        const bool per_n = a.Pg > 1;
        const int64_t wstride = (int64_t)NV * wplane;   // snapshot stride, state pools
        const int64_t rstride = (int64_t)NV * rplane;   // snapshot stride, residual pool
        double dk[P / 2 + 1];   // d_k = D[k][0] (DSHARE)
#pragma unroll
        for (int kk = 1; kk <= P / 2; ++kk) dk[kk] = DSHARE ? S.dmat[kk * P] : 0.0;
        // the loop in two copies, selected once: a run-time per_n inside it made the
        // compiler form the moving-mesh division for every (variable, snapshot)
        auto update = [&](auto per_n_tag) {
            constexpr bool PER_N = decltype(per_n_tag)::value;
            for (int k = 0; k < NV; ++k) {
                const int64_t wo = b.w_off + k * wplane + cell_w, ro = b.r_off + k * rplane + cell_r;
                // W_m of every snapshot first (they feed every n).  LAZY 0: R_n
                // and W^0_n of every snapshot loaded up front as well (3 P values
                // held); 1: W^0_n one snapshot ahead of its use; 2: R_n too (P + 4
                // values held).  W^0_n is always loaded before the store that may
                // replace it (stage 4 writes W^0's slot).
                constexpr int LAZY = VISC ? HBNS_UPDATE_LAZY_VISC : HBNS_UPDATE_LAZY;
                double wm[P], rn[LAZY < 2 ? P : 1], qn[LAZY < 1 ? P : 1];
    #pragma unroll
                for (int m = 0; m < P; ++m) {
                    wm[m] = w[wo + m * wstride];
                    if (LAZY < 2) rn[m] = a.r[ro + m * rstride];
                    if (LAZY < 1) qn[m] = w0[wo + m * wstride];
                }
                double rn_next = LAZY == 2 ? a.r[ro] : 0.0, qn_next = LAZY >= 1 ? w0[wo] : 0.0;
                // sum_m D[n][m] W_m for every n at once when D is circulant and
                // antisymmetric (HBNS_FLAG_D_CIRCULANT): D[m+k][m] = d_k and
                // D[m-k][m] = -d_k bitwise, so one product d_k W_m serves row m + k
                // (added) and row m - k (subtracted) -- (-d) w == -(d w) and
                // s + (-x) == s - x exactly -- and the +0 diagonal term is the zero
                // carrying W_m's sign.  Every row still receives its terms in m
                // ascending order, the first one (m = 0) unadded, as specified.
                double hb[DSHARE ? P : 1];
                if (DSHARE) {
                    hb[0] = hbgpu::zero_times(wm[0]);
    #pragma unroll
                    for (int kk = 1; kk <= P / 2; ++kk) {
                        const double prod = mul(dk[kk], wm[0]);
                        hb[kk] = prod;
                        hb[P - kk] = -prod;
                    }
    #pragma unroll
                    for (int m = 1; m < P; ++m) {
    #pragma unroll
                        for (int kk = 1; kk <= P / 2; ++kk) {
                            const double prod = mul(dk[kk], wm[m]);
                            hb[(m + kk) % P] = add(hb[(m + kk) % P], prod);
                            hb[(m + P - kk) % P] = sub(hb[(m + P - kk) % P], prod);
                        }
                        hb[m] = add(hb[m], hbgpu::zero_times(wm[m]));
                    }
                }
    #pragma unroll
                for (int n = 0; n < P; ++n) {
                    double qn_n, rn_n;
                    if (LAZY >= 1) {
                        qn_n = qn_next;
                        if (n + 1 < P) qn_next = w0[wo + (n + 1) * wstride];
                    } else {
                        qn_n = qn[n];
                    }
                    if (LAZY == 2) {
                        rn_n = rn_next;
                        if (n + 1 < P) rn_next = a.r[ro + (n + 1) * rstride];
                    } else {
                        rn_n = rn[n];
                    }
                    double V = V0, cdt = cdt0;
                    if (PER_N) {
                        V = volc[(int64_t)n * wplane];
                        cdt = dv(mul(coef, dtc), V);
                    }
                    double s;
                    if (DSHARE) {
                        s = hb[n];
                    } else {
                        s = mul(S.dmat[n * P], wm[0]);
    #pragma unroll
                        for (int m = 1; m < P; ++m) s = add(s, mul(S.dmat[n * P + m], wm[m]));
                    }
                    const double R = add(rn_n, mul(V, s));
                    if (first && k == 0) sq = __fma_rn(R, R, sq);
                    const double v = sub(qn_n, mul(cdt, R));
                    w_out[wo + n * wstride] = v;
                    if (!isfinite(v)) {
                        const long long lin = (((long long)(n * NV + k) * b.nj + (cj - 1)) * b.ni) + (ci - 1);
                        atomicMin(a.status + blockIdx.y, hbgpu::divergence_key(gstage, lin));
                    }
                }
            }
        };
        if (per_n) update(std::true_type{});
        else update(std::false_type{});
    }
    // the tile's residual rows are consumed: drop their L2 lines without a
    // write-back (only whole 128-B lines inside this tile's row segments)
#if HBNS_DISCARD
    __syncthreads();
    for (int t = threadIdx.x; t < P * NV * TJ; t += FLUX_THREADS) {
        const int r = t % TJ, k = (t / TJ) % NV, n = t / (TJ * NV);
        if (j0 + r > b.nj) continue;
        const int len = min(TI, b.ni - i0 + 1) * 8;
        const uintptr_t s0 = (uintptr_t)(a.r + rs(b, n, k, j0 + r, i0));
        for (uintptr_t l = (s0 + 127) & ~(uintptr_t)127; l + 128 <= s0 + len; l += 128)
            asm volatile("discard.global.L2 [%0], 128;" ::"l"(l) : "memory");
    }
#endif
    if (first) {
        // stage-1 norm partial of the tile: fixed shuffle tree per warp, warps in order
        for (int o = 16; o > 0; o >>= 1) sq = add(sq, __shfl_down_sync(0xffffffffu, sq, o));
        if (lane == 0) red[warp] = sq;
        __syncthreads();
        if (threadIdx.x == 0) {
            double t = 0.0;
            for (int k = 0; k < NW; ++k) t = add(t, red[k]);
            a.norm_part[b.part_off + tile] = t;
        }
    }
}

// stage-1 norm: one warp per block folds that block's tile partials in a
// fixed lane-strided order and shuffle tree; one thread then folds blocks in
// order
__global__ void ns_norm_kernel(hbns_args a, int iter) {
    __shared__ double blk_sum[1024];
    if (a.iter_dev) iter = *a.iter_dev;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    for (int bk = warp; bk < a.nblocks; bk += nw) {
        const hbns_block &b = a.blocks[bk];
        const int used = ((b.ni + TI - 1) / TI) * ((b.nj + TJ - 1) / TJ);
        double s = 0.0;
        for (int c = lane; c < used; c += 32) s = add(s, a.norm_part[b.part_off + c]);
        for (int o = 16; o > 0; o >>= 1) s = add(s, __shfl_down_sync(0xffffffffu, s, o));
        if (lane == 0) {
            blk_sum[bk] = s;
            if (a.blk_norms) a.blk_norms[(int64_t)iter * a.nglobal + b.gid] = s;
        }
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
    if (a.iter_dev) iter = *a.iter_dev;
    __shared__ double px[FORCE_CHUNK], py[FORCE_CHUNK];
    __shared__ int seg_bs[MAX_WALL_SEGS], seg_end[MAX_WALL_SEGS];   // block * 4 + side, running end
    __shared__ int seg_gpos[MAX_WALL_SEGS];                            // job-wide position of its first face
    __shared__ int nseg_s;
    const int n = blockIdx.x;
    const int g = a.Pg > 1 ? n : 0;
    if (threadIdx.x == 0) {
        int ns = 0, end = 0;
        for (int bk = 0; bk < a.nblocks && ns < MAX_WALL_SEGS; ++bk) {
            const hbns_block &b = a.blocks[bk];
            int gpos = b.wall_off;
            for (int side = 0; side < 4; ++side) {
                if (b.kinds[side] != HBNS_NOSLIP && b.kinds[side] != HBNS_SLIP) continue;
                const int len = side < 2 ? b.ni : b.nj;
                end += len;
                seg_bs[ns] = bk * 4 + side;
                seg_end[ns] = end;
                seg_gpos[ns] = gpos;
                gpos += len;
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
            if (a.wall_prod) {   // multi-rank: the products at their job-wide positions
                const int64_t pos = seg_gpos[sg] + e - 1;
                a.wall_prod[((int64_t)iter * a.P + n) * 2 * a.nwall + pos] = mul(q.p, sx);
                a.wall_prod[(((int64_t)iter * a.P + n) * 2 + 1) * a.nwall + pos] = mul(q.p, sy);
                continue;
            }
            px[t - c0] = mul(q.p, sx);
            py[t - c0] = mul(q.p, sy);
        }
        if (a.wall_prod) continue;
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

// job-wide wall forces of a multi-rank run: one thread per (iteration,
// snapshot), the specification's left-to-right folds over the summed products
__global__ void ns_wall_fold_kernel(const double *prod, int iters, int P, int nwall, double *forces) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= iters * P) return;
    const double *px = prod + (int64_t)t * 2 * nwall, *py = px + nwall;
    double fx = 0.0, fy = 0.0;
    for (int f = 0; f < nwall; ++f) {
        fx = add(fx, px[f]);
        fy = add(fy, py[f]);
    }
    forces[(int64_t)t * 2] = fx;
    forces[(int64_t)t * 2 + 1] = fy;
}

// the device iteration counter (graph replays): advanced after the forces
__global__ void ns_iter_advance_kernel(int32_t *iter) { *iter += 1; }

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

template <bool VISC, int P, int MINB, bool DSHARE>
static int stage_launch_kd(const hbns_args *a, int32_t slot_in, int32_t slot_out, double coef, int first, int iter,
                          int64_t tiles, cudaStream_t s) {
    static bool ready[hbgpu::HB_MAX_DEVICES];
    const int dev = hbgpu::current_device();
    if (dev < 0) return HBGPU_ERR_CUDA;
    const size_t smem = sizeof(FluxSmem);
    if (!ready[dev]) {
        if (cudaFuncSetAttribute(ns_stage_kernel<VISC, P, MINB, DSHARE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem) != cudaSuccess)
            return check("hbns_stage (smem attribute)");
        ready[dev] = true;
    }
    ns_stage_kernel<VISC, P, MINB, DSHARE><<<dim3((unsigned)tiles, a->nblocks), FLUX_THREADS, smem, s>>>(
        *a, a->w[slot_in], a->w[0], a->w[slot_out], coef, first, iter);
    return HBGPU_OK;
}

template <bool VISC, int P, int MINB>
static int stage_launch_k(const hbns_args *a, int32_t slot_in, int32_t slot_out, double coef, int first, int iter,
                          int64_t tiles, cudaStream_t s) {
    if (a->flags & HBNS_FLAG_D_CIRCULANT)
        return stage_launch_kd<VISC, P, MINB, true>(a, slot_in, slot_out, coef, first, iter, tiles, s);
    return stage_launch_kd<VISC, P, MINB, false>(a, slot_in, slot_out, coef, first, iter, tiles, s);
}

// CTAs per SM the kernel variant is compiled for.  Viscous: 2 (96 registers).
// Euler: 3 (72 registers) on a grid of many waves -- C4: 170 vs 187 ms per
// iteration -- but 2 (96 registers, fewer spills: a tile takes ~0.73 of the
// time) when the grid is so small that both fill the same number of waves --
// C2, 512 tiles: 0.58 vs 0.71 ms.  The rule compares waves x tile time.
template <bool VISC, int P>
static int stage_launch(const hbns_args *a, int32_t slot_in, int32_t slot_out, double coef, int first, int iter,
                        cudaStream_t s) {
    const int64_t tiles = (int64_t)((a->max_ni + TI - 1) / TI) * ((a->max_nj + TJ - 1) / TJ);
#ifdef HBNS_FLUX_MINB
    return stage_launch_k<VISC, P, HBNS_FLUX_MINB>(a, slot_in, slot_out, coef, first, iter, tiles, s);
#else
    if constexpr (VISC) {
        return stage_launch_k<VISC, P, 2>(a, slot_in, slot_out, coef, first, iter, tiles, s);
    } else {
        static int sms[hbgpu::HB_MAX_DEVICES];
        const int dev = hbgpu::current_device();
        if (dev < 0) return HBGPU_ERR_CUDA;
        if (sms[dev] == 0 && cudaDeviceGetAttribute(&sms[dev], cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
            return check("hbns_stage (SM count)");
        const int64_t total = tiles * a->nblocks;
        const int64_t waves3 = (total + 3 * sms[dev] - 1) / (3 * sms[dev]), waves2 = (total + 2 * sms[dev] - 1) / (2 * sms[dev]);
        if (0.733 * (double)waves2 < (double)waves3)
            return stage_launch_k<VISC, P, 2>(a, slot_in, slot_out, coef, first, iter, tiles, s);
        return stage_launch_k<VISC, P, 3>(a, slot_in, slot_out, coef, first, iter, tiles, s);
    }
#endif
}

template <bool VISC>
static int stage_dispatch(const hbns_args *a, int32_t slot_in, int32_t slot_out, double coef, int first, int iter,
                          cudaStream_t s) {
    switch (a->P) {
        case 1: return stage_launch<VISC, 1>(a, slot_in, slot_out, coef, first, iter, s);
        case 3: return stage_launch<VISC, 3>(a, slot_in, slot_out, coef, first, iter, s);
        case 5: return stage_launch<VISC, 5>(a, slot_in, slot_out, coef, first, iter, s);
        case 7: return stage_launch<VISC, 7>(a, slot_in, slot_out, coef, first, iter, s);
        case 9: return stage_launch<VISC, 9>(a, slot_in, slot_out, coef, first, iter, s);
        default: break;
    }
    hbgpu_set_error("hbns_stage: P = %d not templated (1..9 odd)", a->P);
    return HBGPU_ERR_UNSUPPORTED;
}

extern "C" int hbns_stage(const hbns_args *a, int32_t slot_in, int32_t slot_out, double coef, int32_t iter,
                          int32_t first, void *stream) {
    if (a == nullptr || slot_in < 0 || slot_in > 2 || slot_out < 0 || slot_out > 2 || a->max_ni < 1 ||
        a->max_nj < 1) {
        hbgpu_set_error("hbns_stage: bad arguments");
        return HBGPU_ERR_ARG;
    }
    const int64_t tiles = (int64_t)((a->max_ni + TI - 1) / TI) * ((a->max_nj + TJ - 1) / TJ);
    if (tiles > INT32_MAX || a->nblocks > 1024) {
        hbgpu_set_error("hbns_stage: grid too large (%lld tiles, %d blocks)", (long long)tiles, a->nblocks);
        return HBGPU_ERR_ARG;
    }
    cudaStream_t s = (cudaStream_t)stream;
    if (a->stage < 0 || a->stage > 3) {
        hbgpu_set_error("hbns_stage: args->stage %d is not an RK stage (0..3)", a->stage);
        return HBGPU_ERR_ARG;
    }
    int rc = a->mu > 0.0 ? stage_dispatch<true>(a, slot_in, slot_out, coef, first != 0, iter, s)
                         : stage_dispatch<false>(a, slot_in, slot_out, coef, first != 0, iter, s);
    if (rc) return rc;
    int n = 1;
    if (first) {
        ns_norm_kernel<<<1, 1024, 0, s>>>(*a, iter);
        ++n;
    }
    hbgpu_count_launch(n);
    return check("hbns_stage");
}

extern "C" int hbns_wall_fold(const double *wall_prod, int32_t iters, int32_t P, int32_t nwall, double *forces,
                              void *stream) {
    if (iters <= 0 || P <= 0) return HBGPU_OK;
    if (wall_prod == nullptr || forces == nullptr || nwall < 0) {
        hbgpu_set_error("hbns_wall_fold: bad arguments");
        return HBGPU_ERR_ARG;
    }
    ns_wall_fold_kernel<<<(iters * P + 127) / 128, 128, 0, (cudaStream_t)stream>>>(wall_prod, iters, P, nwall, forces);
    hbgpu_count_launch(1);
    return check("hbns_wall_fold");
}

extern "C" int hbns_forces(const hbns_args *a, int32_t iter, void *stream) {
    if (a->nblocks > 256) {
        hbgpu_set_error("hbns_forces: at most 256 blocks");
        return HBGPU_ERR_ARG;
    }
    ns_forces_kernel<<<a->P, FORCE_THREADS, 0, (cudaStream_t)stream>>>(*a, a->w[0], iter);
    if (a->iter_dev) {
        ns_iter_advance_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(a->iter_dev);
        hbgpu_count_launch(1);
    }
    hbgpu_count_launch(1);
    return check("hbns_forces");
}
