/*
 * hbns.h -- C ABI of the north-star HB Euler / laminar Navier-Stokes stage
 * in libhbgpu.so.  The reference (hbproxy) has no flux
 * physics (hbcore.py:3-13), so these entry points replace no
 * reference function; they implement the specification in
 * paper_1304_7654_b200/nsflow.py and are checked against the builder-written
 * oracle/ns_oracle.c (parity unpinned).
 *
 * One RK stage of the host loop (nsflow.NSRun):
 *   cut halos (hbgpu_halo, two layers) -> hbns_boundaries(slot_in)
 *   -> hbns_stage(slot_in, slot_out, alpha_s)
 * and after the fourth stage hbns_forces.  All pointers are device memory
 * except the args struct itself; every call is asynchronous on `stream`.
 */
#ifndef HBNS_H
#define HBNS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HBNS_FARFIELD 0
#define HBNS_NOSLIP 1
#define HBNS_SLIP 2
#define HBNS_CUT 3

/* hbns_stage tiles: HBNS_TILE_I columns x HBNS_TILE_J rows of a block per
 * CTA; norm_part holds one partial per tile (part_off per block)          */
#define HBNS_TILE_I 32
#define HBNS_TILE_J 8

typedef struct hbns_block {
    int64_t w_off;       /* element offset of the block in every state pool   */
    int64_t r_off;       /* ... in the residual pool (P, 4, nj, ni)            */
    int64_t dt_off;      /* ... in the time-step pool (nj, ni)                 */
    int64_t c_off;       /* ... in the cell-geometry pools (Pg, nj+4, ni+4)    */
    int64_t fi_off;      /* ... in the i-face pools (Pg, nj+4, ni+5)           */
    int64_t fj_off;      /* ... in the j-face pools (Pg, nj+5, ni+4)           */
    int64_t part_off;    /* ... in the stage-1 norm partials (one per tile)   */
    int32_t ni, nj;
    int32_t kinds[4];    /* south, north, west, east: HBNS_*                   */
    int32_t gid;         /* index of the block in the job (ids ascending)      */
    int32_t wall_off;    /* position of its first wall face in the job's wall
                            order (blocks ascending, sides S/N/W/E, cells)    */
} hbns_block;

#define HBNS_FLAG_D_CIRCULANT 1

typedef struct hbns_args {
    double *w[3];                /* state slots: 0 = iteration start         */
    double *r;                   /* residual pool                             */
    double *dt;                  /* local time steps                          */
    const double *xc, *yc, *vol; /* cell geometry                             */
    const double *six, *siy, *gi;/* i-face normals, grid flux (moving)        */
    const double *sjx, *sjy, *gj;/* j-face normals, grid flux (moving)        */
    const hbns_block *blocks;
    const double *winf;          /* freestream state per snapshot (P x 4)     */
    const double *dmat;          /* HB matrix D (P x P)                       */
    unsigned long long *status;  /* per block: first non-finite key, ~0 none  */
    double *norm_part;           /* stage-1 partials                          */
    double *norms;               /* per iteration                             */
    double *forces;              /* per iteration, snapshot: (fx, fy)         */
    /* multi-rank runs (else null): per iteration the per-block sums of
     * R_rho^2 at [iter * nglobal + gid], and the wall-face products p S at
     * [((iter * P + n) * 2 + xy) * nwall + position]; summed over the ranks
     * they fold (hbgpu_norm_totals, hbns_wall_fold) exactly as one rank's    */
    double *blk_norms;
    double *wall_prod;
    /* non-null: the iteration index is read from this device counter (the
     * `iter` arguments are ignored) and hbns_forces advances it, so one
     * captured iteration replays as the next                               */
    int32_t *iter_dev;
    double mu, cfl, omega_nh;    /* M/Re (0: Euler), CFL, omega * N_H         */
    double kq;                   /* (mu * gamma) / Pr, as the host rounds it  */
    int32_t nblocks, P, Pg, moving;
    int32_t max_len, max_cells;  /* largest block side, largest ni * nj       */
    int32_t max_ni, max_nj;      /* largest ni, largest nj (residual grid)    */
    int32_t nglobal, nwall;      /* blocks / wall faces of the whole job      */
    int32_t stage, flags;        /* RK stage (0..3) of the next hbns_stage:
                                    status keys are ((iter*4 + stage + 1) << 40)
                                    | (n, k, j, i) index, an atomicMin keeps the
                                    first offending stage, then cell          */
    /* flags: HBNS_FLAG_D_CIRCULANT (1) = dmat is bitwise circulant and
     * antisymmetric with a +0 diagonal, as the reference's spectral_matrix
     * (hbcore.py:88-94) is: the update then multiplies by the N_H constants
     * D[k][0] and shares each product between rows m + k and m - k -- the
     * same values, as (-d) w == -(d w) and s + (-x) == s - x in IEEE
     * arithmetic.  Only set it after checking the matrix on the host.       */
} hbns_args;

int hbns_boundaries(const hbns_args *a, int32_t slot, void *stream);
/* One RK stage: residual of slot_in (halos filled), HB source, update
 * W(slot_out) = W(slot 0) - (coef dt / V) R.  first != 0 (stage 1, slot_in
 * = 0): the local time step is formed from slot 0 into `dt` first, and the
 * residual norm of iteration `iter` is written to norms[iter].            */
int hbns_stage(const hbns_args *a, int32_t slot_in, int32_t slot_out, double coef, int32_t iter,
               int32_t first, void *stream);
int hbns_forces(const hbns_args *a, int32_t iter, void *stream);
/* forces[(it * P + n) * 2 + xy] = left-to-right sum over the nwall faces of
 * wall_prod[((it * P + n) * 2 + xy) * nwall + f], it < iters               */
int hbns_wall_fold(const double *wall_prod, int32_t iters, int32_t P, int32_t nwall, double *forces,
                   void *stream);

#ifdef __cplusplus
}
#endif

#endif /* HBNS_H */
