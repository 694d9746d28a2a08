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
 *   -> [stage 1: hbns_timestep(slot 0)] -> hbns_residual(slot_in)
 *   -> hbns_update(slot_in, slot_out, alpha_s)
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

typedef struct hbns_block {
    int64_t w_off;       /* element offset of the block in every state pool   */
    int64_t r_off;       /* ... in the residual pool (P, 4, nj, ni)            */
    int64_t dt_off;      /* ... in the time-step pool (nj, ni)                 */
    int64_t c_off;       /* ... in the cell-geometry pools (Pg, nj+4, ni+4)    */
    int64_t fi_off;      /* ... in the i-face pools (Pg, nj+4, ni+5)           */
    int64_t fj_off;      /* ... in the j-face pools (Pg, nj+5, ni+4)           */
    int64_t part_off;    /* ... in the stage-1 norm partials (P * ctas)        */
    int32_t ni, nj;
    int32_t kinds[4];    /* south, north, west, east: HBNS_*                   */
} hbns_block;

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
    unsigned long long *status;  /* per block: first non-finite lin, ~0 none  */
    double *norm_part;           /* stage-1 partials                          */
    double *norms;               /* per iteration                             */
    double *forces;              /* per iteration, snapshot: (fx, fy)         */
    double mu, cfl, omega_nh;    /* M/Re (0: Euler), CFL, omega * N_H         */
    double kq;                   /* (mu * gamma) / Pr, as the host rounds it  */
    int32_t nblocks, P, Pg, moving;
    int32_t max_len, max_cells;  /* largest block side, largest ni * nj       */
    int32_t max_ni, max_nj;      /* largest ni, largest nj (residual grid)    */
} hbns_args;

int hbns_boundaries(const hbns_args *a, int32_t slot, void *stream);
int hbns_timestep(const hbns_args *a, int32_t slot, void *stream);
int hbns_residual(const hbns_args *a, int32_t slot, void *stream);
int hbns_update(const hbns_args *a, int32_t slot_in, int32_t slot_out, double coef, int32_t iter,
                int32_t want_norm, void *stream);
int hbns_forces(const hbns_args *a, int32_t iter, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* HBNS_H */
