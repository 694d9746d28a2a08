/*
 * hbgpu.h -- C ABI of the B200-native HB residual-and-smoothing library
 * (libhbgpu.so, built from paper_1304_7654_b200/csrc/).
 *
 * Plain pointers, sizes and a cudaStream_t passed as void*; no torch types.
 * Every function returns 0 on success and a nonzero hbgpu status otherwise;
 * hbgpu_last_error() describes the last failure on the calling thread.
 * All device pointers are caller-owned; the library never allocates device
 * memory except the CUDA graph it may instantiate inside an engine.
 *
 * Each entry point names the reference interface it replaces (file:line
 * under /root/reference/pkg/src/hbproxy/).
 */
#ifndef HBGPU_H
#define HBGPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HBGPU_ABI_VERSION 2
#define HBGPU_NPDE 4
/* largest snapshot count handled by the register-window stage kernels;
 * larger P runs the generic kernel */
#define HBGPU_MAX_TEMPLATED_P 17
/* largest snapshot count of the library (forcing amplitudes travel as a
 * kernel parameter of HBGPU_MAX_P*4 doubles) */
#define HBGPU_MAX_P 127
/* largest snapshot count of the paired-stage kernel (shared-memory bound) */
#define HBGPU_MAX_PAIR_P 9
/* elements of the device row lead: cell i (0 = west halo) of row j sits at
 * row_base + HBGPU_ROW_LEAD + i, so interior cell i=1 -- and every stage
 * strip -- starts on a 64-byte DRAM access granule (rows are padded to a
 * multiple of 8 doubles) */
#define HBGPU_ROW_LEAD 7
/* consumer warps per stage tile (= residual-norm partials per tile).  A
 * tile covers tile_pdes pdes (4 or 1) and 256 / tile_pdes columns: each of
 * the 8 warps owns 32 columns of one pde. */
#define HBGPU_TILE_WARPS 8
/* interior columns per strip for tile_pdes = 4 (the narrow-block default) */
#define HBGPU_STRIP 64

enum {
    HBGPU_OK = 0,
    HBGPU_ERR_CUDA = 1,
    HBGPU_ERR_ARG = 2,
    HBGPU_ERR_NCCL = 3,
    HBGPU_ERR_UNSUPPORTED = 4
};

/* ---- device data layout -------------------------------------------------
 * A "slot" is one device allocation holding the full state of every block a
 * rank owns.  Block b's value (n, p, j, i) -- plane n, pde p, array row j in
 * [0, nj+1], array column i in [0, ni+1] -- lives at element
 *     base + (n*4 + p)*ps + j*rs + HBGPU_ROW_LEAD + i
 * of the slot.  Three slots rotate through the RK stages.  Two layouts:
 * plane-major (ps = (nj+2)*pitch, rs = pitch) and row-interleaved
 * (ps = pitch, rs = 4*P*pitch: row j of all (n, p) planes contiguous).     */
typedef struct hbgpu_block {
    int64_t base;        /* element offset of (0,0,0,-LEAD) in every slot   */
    int64_t ps;          /* elements between consecutive (n, p) planes      */
    int64_t rs;          /* elements between consecutive rows j            */
    int32_t ni, nj;      /* interior cells                                  */
    int32_t pitch;       /* row stride, elements (multiple of 8)            */
    int32_t gid;         /* global block id                                 */
    int32_t tiles_i;     /* column strips: ceil(ni / (256 / tile_pdes))     */
    int32_t tiles_j;     /* ceil(nj / tile_rows)                            */
    int32_t tile_begin;  /* first tile of this block in the rank tile list  */
    int32_t ntiles;      /* tiles_i * (4 / tile_pdes) * tiles_j; tile t of
                            the block: strip t % tiles_i, pde group
                            (t / tiles_i) % (4 / tile_pdes), row tile rest  */
    int32_t sxy_pitch;   /* row stride of the sxy table (ni rounded up to 4) */
    int32_t pad0;
    double nu_h2;        /* NU / (h*h)          (hbcore.py:257)             */
    double adv_2h;       /* ADVECTION / (2*h)   (hbcore.py:257)             */
    double h;
    int64_t sxy_off;     /* element offset of the block's sxy table (32-B aligned,
                            nj rows of sxy_pitch)                        */
    int64_t face_off[4]; /* entry offset into the face-target pool per face
                            (south, north, west, east), -1 = no cut cell    */
} hbgpu_block;

/* Halo target of one interior face cell (fused halo forwarding):
 *   ps >  0 : local halo cell, element `off` of the output slot at (n,p)=(0,0),
 *             stride ps between (n,p) planes;
 *   ps == 0 : no target (non-cut boundary cell);
 *   ps <  0 : remote, send-buffer element off + n*4 + p (element-major,
 *             exchange.py:248-252).                                        */
typedef struct hbgpu_face_target {
    int64_t off;         /* bit HBGPU_SECTOR_TARGET_BIT set (local targets):
                            the cell's 32-byte sector holds no other cell of
                            the block, so it may be written as a whole      */
    int64_t ps;
} hbgpu_face_target;
#define HBGPU_SECTOR_TARGET_BIT 62

/* Divergence status keys (hbgpu_stage_args.status, one per block, reset to
 * all-ones; kernels atomicMin into them):
 *   (gstage << 40) | lin        a non-finite value at global stage gstage
 *                               (iteration*4 + stage + 1), lin = the
 *                               lexicographic (n, p, j-1, i-1) interior
 *                               index (hbcore.py:279-284)
 *   ... | HBGPU_HAZARD_BIT      a finite value of magnitude >= 2^1022 (the
 *                               paired kernel's exact rewrites need
 *                               |q| < 2^1022; the host then repeats the
 *                               run on the strict single-stage kernels)   */
#define HBGPU_STATUS_LIN_BITS 40
#define HBGPU_HAZARD_BIT (1ull << 39)

/* One halo copy direction for the standalone halo kernel (priming exchange,
 * unpack after a receive, exchange_halos).  Value v = n*4 + p of element e
 * moves from src_base[src_off + e*src_es + v*src_vs] to
 * dst_base[dst_off + e*dst_es + v*dst_vs]; `src_kind`/`dst_kind` select the
 * base: 0 = the state slot, 1 = send buffer, 2 = receive buffer.           */
typedef struct hbgpu_halo_dir {
    int64_t src_off, src_es, src_vs;
    int64_t dst_off, dst_es, dst_vs;
    int32_t length;
    int32_t src_kind, dst_kind;
    int32_t flags;       /* HBGPU_HALO_SECTOR_DST: every destination cell's
                            32-byte sector holds no other live value (a
                            west halo column; an east one when ni % 4 == 0),
                            so it is written as a whole sector            */
} hbgpu_halo_dir;
#define HBGPU_HALO_SECTOR_DST 1

/* Force-integration segment: one (block, face) body face, in reference
 * order (blocks ascending, body_faces order; hbcore.py:369-381).          */
typedef struct hbgpu_force_seg {
    int64_t start;       /* element offset of face cell 1 at (n,p)=(0,0)   */
    int64_t stride;      /* elements between consecutive face cells        */
    int64_t ps;          /* elements between (n, p) planes                 */
    int32_t length;      /* face extent                                    */
    int32_t body;
    double h;
} hbgpu_force_seg;

/* Remote transfer of one cut direction (NCCL send or receive). */
typedef struct hbgpu_peer_msg {
    int32_t peer;        /* rank */
    int32_t pad;
    int64_t offset;      /* element offset in the send / receive buffer     */
    int64_t count;       /* doubles                                        */
} hbgpu_peer_msg;

/* ---- kernel-level drop-ins (reference dense layout) ----------------------
 * q/q0: (planes, npde, nj2, ni2) C-order fp64; resid/src: (planes, npde,
 * nj2-2, ni2-2).  Bounds are the reference's array coordinates.           */

/* replaces hbcore._residual_kernel (hbcore.py:184-221) */
int hbgpu_residual(const double *q, const double *dmat, const double *src,
                   double nu_h2, double adv_2h, double *out,
                   int64_t planes, int64_t npde, int64_t nj2, int64_t ni2,
                   int64_t n_lo, int64_t n_hi, int64_t j_lo, int64_t j_hi,
                   void *stream);

/* replaces hbcore._update_kernel (hbcore.py:224-245).  Instead of the
 * poisoned accumulator the kernel atomically lowers *first_bad (device,
 * initialise to UINT64_MAX) to the linear interior index
 * ((n*npde + p)*nj + (j-1))*ni + (i-1) of any non-finite value it writes. */
int hbgpu_update(double *q, double *q0, const double *resid, double coef,
                 int snapshot, int64_t planes, int64_t npde, int64_t nj2,
                 int64_t ni2, int64_t n_lo, int64_t n_hi, int64_t j_lo,
                 int64_t j_hi, unsigned long long *first_bad, void *stream);

/* replaces the np.argwhere scan of hbcore._raise_divergence (hbcore.py:279-284):
 * lowers *first_bad to the first non-finite interior value of q.          */
int hbgpu_first_nonfinite(const double *q, int64_t planes, int64_t npde,
                          int64_t nj2, int64_t ni2,
                          unsigned long long *first_bad, void *stream);

/* ---- production kernels on the slot layout ------------------------------ */

typedef struct hbgpu_stage_args {
    const double *in;          /* slot read by the stencil (q_{s-1})       */
    const double *q0;          /* slot holding the iteration start (q_0)   */
    double *out;               /* slot written (q_s), may equal q0         */
    const double *band;        /* pair != 0: the band slot (slot 2)        */
    double *sendbuf;           /* remote halo payloads (may be NULL)       */
    const hbgpu_block *blocks; /* device array [nblocks]                   */
    const int32_t *tile_block;  /* device array [total_tiles]: tile -> block */
    const double *sxy;         /* device forcing tables                    */
    const hbgpu_face_target *faces; /* device face-target pool             */
    double *norm_part;         /* device [total_tiles * HBGPU_TILE_WARPS]
                                  (stage 0) or NULL                         */
    unsigned long long *status;/* device [nblocks] divergence keys         */
    const int32_t *iter;       /* device iteration counter                 */
    const double *dmat;        /* device P*P (generic kernel only)         */
    const void *tmaps;         /* device [HBGPU_TMAP_SETS][nblocks]
                                  CUtensorMap (hbgpu_encode_tensor_maps)    */
    int32_t nblocks;
    int32_t total_tiles;
    int32_t planes;
    int32_t stage;             /* 0..3                                      */
    int32_t tile_rows;
    int32_t in_slot;           /* which of the three slots `in` is (0..2);
                                  q0 is slot 0                              */
    int32_t interleaved;       /* 1 = row-interleaved slot layout          */
    int32_t tile_pdes;         /* pdes per tile: 4 (64-col strips) or 1
                                  (256-col strips)                          */
    int32_t out_slot;          /* which of the three slots `out` is (0..2) */
    int32_t pair;              /* 0: one stage.  1 / 2: two stages fused
                                  (s, s+1) = (0, 1) / (2, 3): the first
                                  stage's values at the tile perimeters come
                                  from the band slot (hbgpu_band), slot 2  */
    double coef;               /* alpha_s * dtau                            */
    double coef2;              /* alpha_{s+1} * dtau (pair != 0)            */
    const struct hbgpu_band_seg *band_segs; /* hbgpu_band: device segments  */
    int32_t nband_segs;
    int32_t band_max_len;
    /* pair != 0: device [total_tiles * tile_rows * 2 * tile_pdes * planes].
     * Pass A (pair 1) saves q0 at each tile's strip-edge columns inside the
     * block; pass B (pair 2), which overwrites q0 in place, reads them back
     * from here: by then the neighbouring strip's CTA may have replaced q0
     * at those columns                                                      */
    double *edge_q0;
    /* tiles this launch processes: tile_order[k] (identity when NULL) for k
     * in [tile_lo, tile_hi), tile_hi <= 0 meaning total_tiles.  The engine
     * splits a multi-GPU stage into its boundary tiles (whose faces feed a
     * remote cut) and the interior tiles that overlap the NCCL exchange.  */
    const int32_t *tile_order;
    int32_t tile_lo;
    int32_t tile_hi;
    /* D row-major P x P with a +0.0 diagonal (hbcore.py:88-94); ap[n*4 + p]
     * = amp[n] (1 + p/4), zero except on planes 1 and 2 (hbcore.py:170-175):
     * the kernel adds those zero terms as exact signed zeros              */
    double D[HBGPU_MAX_TEMPLATED_P * HBGPU_MAX_TEMPLATED_P];
    double ap[HBGPU_MAX_P * HBGPU_NPDE];
} hbgpu_stage_args;

/* A run of tile-perimeter cells for hbgpu_band: `len` cells of block
 * `block` from array cell (j, i) along a row (dir 0) or a column (dir 1). */
typedef struct hbgpu_band_seg {
    int32_t block;       /* local block index */
    int32_t dir;
    int32_t j, i;
    int32_t len;
    int32_t pad;
} hbgpu_band_seg;

/* One RK stage (args->stage, args->coef) at the listed cells only: the
 * values the paired stage kernel (args->pair != 0) reads outside its tile.
 * Writes them into args->out (the band slot) at their own cells and forwards
 * cut-face cells into the band slot's halos / the send buffer, with the
 * reference's rounding (hbcore.py:184-245) and divergence keys.            */
int hbgpu_band(const hbgpu_stage_args *args, void *stream);

/* one fused RK stage over every owned block: residual (hbcore.py:184-221),
 * update (hbcore.py:224-245), local halo forwarding and remote pack
 * (exchange.py:248-261), divergence keys, residual-norm partials */
int hbgpu_stage(const hbgpu_stage_args *args, void *stream);

/* resolve kernel attributes / occupancy for a snapshot count ahead of any
 * CUDA graph capture (hbgpu_engine_create calls it) */
int hbgpu_stage_prepare(int32_t planes);

/* 1 when the first RK stage of the single-stage schedule (args->stage == 0,
 * args->pair == 0) forwards its own west / east face columns for this
 * snapshot count, as stages 1..3 always do; 0 when a column-halo pass
 * (hbgpu_halo over the post directions) must follow that launch.  The
 * reference exchanges every face after every stage (exchange.py:295-316);
 * this only says which launch moves the column faces. */
int hbgpu_stage_first_forwards(int32_t planes);

/* TMA descriptors for the stage kernel: 4-D tensor maps (columns, rows,
 * pde, plane) over each block's part of a slot, written as CUtensorMap
 * (128 B) #(set*nblocks + b) into out_host (caller uploads it to device
 * memory, 64-B aligned): sets 0..2 = stencil boxes (strip + 2 halo columns
 * each side, split in two boxes when wider than TMA's 256) over slot[0..2],
 * set 3 = strip-wide q0 box over slot[0], set 4 = 2-D (column, row)
 * strip-wide box over the block's sxy forcing table, sets 5..7 = strip-wide
 * store boxes over slot[0..2] whose column extent ends at cell ni (the
 * store clips the strip's columns past the block and never touches the
 * halo ring), set 8 = strip-wide row box over slot[2] (the band slot), set
 * 9 = one 64-byte column granule over slot[2] (a strip's edge columns).  tile_pdes (4 or 1) fixes the strip geometry.
 * out_bytes >= HBGPU_TMAP_SETS*nblocks*128.                                 */
#define HBGPU_TMAP_SETS 10
int hbgpu_encode_tensor_maps(double *const slot[3], const double *sxy,
                             const hbgpu_block *blocks_host,
                             int32_t nblocks, int32_t planes, int32_t tile_pdes,
                             void *out_host, int64_t out_bytes);

/* standalone halo moves (exchange.py:295-316 local copy / pack / unpack) */
int hbgpu_halo(double *slot, double *sendbuf, const double *recvbuf,
               const hbgpu_halo_dir *dirs, int32_t ndirs, int32_t max_len,
               int32_t planes, void *stream);

/* per-block sums of the stage-0 norm partials -> sumsq[iter*nblocks + b] */
/* hazard key at gstage 0 for every block whose region of `slot` holds a
 * finite value of magnitude >= 2^1022 (the engine runs it before the
 * priming exchange of a paired-schedule run)                               */
int hbgpu_hazard_scan(const double *slot, const hbgpu_block *blocks, int32_t nblocks,
                      int32_t planes, unsigned long long *status, void *stream);

/* per-iteration residual norms: norms[it] = sqrt(sum over b ascending of
 * sumsq[it * nblocks + b]), one strict left-to-right fold per iteration
 * (the host fold of SURVEY.md §8 a14, bitwise)                             */
int hbgpu_norm_totals(const double *sumsq, int32_t iters, int32_t nblocks, double *norms,
                      void *stream);

int hbgpu_norm_fold(const hbgpu_block *blocks, int32_t nblocks,
                    const double *norm_part, double *sumsq,
                    const int32_t *iter, int32_t max_iters, void *stream);

/* per-rank force partials (hbcore.py:359-382) into
 * hist[iter][k][n][body] (k = cl, cd, cm), then iter += 1.  `max_iters` is
 * hist's capacity in iterations (and sumsq's in hbgpu_norm_fold): a device
 * counter at or past it writes nothing.                                  */
int hbgpu_forces(const double *slot, const hbgpu_force_seg *segs,
                 int32_t nsegs, int32_t planes, int32_t nbody, double *hist,
                 int32_t *iter, int32_t max_iters, void *stream);

/* rank-ordered sum (runtime.py:290-294): out[k] = in[0][k] + in[1][k] + ...
 * over `nranks` stacked buffers of `count` doubles                        */
int hbgpu_ordered_fold(const double *stacked, int32_t nranks, int64_t count,
                       double *out, void *stream);

/* ---- output records (outio.py:79-123 layout, 221-241 writer) ------------
 * One record of a restart or flowtec file: a 4-byte little-endian length
 * prefix (payload bytes), the float64 payload, the same 4-byte suffix.
 * Restart payload of (block, plane n): q[n][p][j][i] for j rows outer, i
 * columns, p innermost (the interior only).  Flowtec payload: per cell
 * (x_i, y_j, q[n][0][j][i], q[n][1][j][i]), rows outer.                     */
enum { HBGPU_RECORD_RESTART = 0, HBGPU_RECORD_FLOWTEC = 1 };

typedef struct hbgpu_out_record {
    int32_t block;    /* local block index into the blocks table            */
    int32_t plane;    /* HB snapshot n                                       */
    int32_t kind;     /* HBGPU_RECORD_RESTART or HBGPU_RECORD_FLOWTEC        */
    int32_t pad;
    int64_t dst;      /* byte offset of the record's length prefix in dst    */
    int64_t xy;       /* flowtec: element offset of the block's x centres
                         (ni values) followed by its y centres (nj) in xy    */
} hbgpu_out_record;

/* Write `nrecs` records (markers + payload, byte-exact file images) from a
 * slot into dst (device memory; records may be 4-byte aligned only).      */
int hbgpu_pack_records(const double *slot, const hbgpu_block *blocks,
                       const hbgpu_out_record *recs, int32_t nrecs,
                       int32_t max_cells, const double *xy, void *dst,
                       void *stream);

/* ---- engine: the per-rank iteration schedule (driver.py:110-149) -------- */

typedef struct hbgpu_engine_desc {
    double *slot[3];                 /* A (q0 / result), B, C              */
    double *sendbuf, *recvbuf;
    const hbgpu_block *blocks;       /* device */
    const int32_t *tile_block;        /* device */
    const double *sxy;               /* device */
    const hbgpu_face_target *faces;  /* device */
    const double *dmat;              /* device */
    double *norm_part;               /* device [total_tiles * HBGPU_TILE_WARPS] */
    double *sumsq;                   /* device [max_iters * nblocks] */
    unsigned long long *status;      /* device [nblocks] */
    int32_t *iter;                   /* device, 1 element */
    const hbgpu_halo_dir *prime_dirs;  int32_t nprime;  int32_t prime_max_len;
    const hbgpu_halo_dir *unpack_dirs; int32_t nunpack; int32_t unpack_max_len;
    /* after the first stage: forwarding of west / east face columns (local
     * halo copies and remote packs).  Inside the stage kernel the consumer
     * warps forward south / north rows and, in the update stages, the TMA
     * store warp forwards west / east columns from the staged row; both use
     * the face-target pool                                                  */
    const hbgpu_halo_dir *post_dirs;   int32_t npost;   int32_t post_max_len;
    /* fused != 0: each iteration runs band(0), pair(0,1), band(2), pair(2,3)
     * and a full halo pass instead of four single stages; slot 2 holds the
     * band values (hbgpu_band), band_segs lists the tile-perimeter cells   */
    const hbgpu_band_seg *band_segs;   int32_t nband_segs; int32_t band_max_len;
    int32_t fused;
    /* small != 0 (single-rank, no remote cut, not fused): hbgpu_engine_iterate
     * runs whole iterations in one cooperative launch (hb_small.cu) instead
     * of the per-stage kernels; small_max_cells = the largest block's
     * ni * nj (sizes the grid)                                              */
    int32_t small;
    double *edge_q0;                 /* fused: device, see hbgpu_stage_args */
    /* multi-GPU overlap (used when comm != NULL and the rank sends): device
     * tile permutation with the nbound_tiles boundary tiles first;
     * prime_dirs / post_dirs start with prime_remote / post_remote remote
     * packs (dst_kind 1), followed by the local copies                    */
    const int32_t *tile_order;
    int32_t nbound_tiles, prime_remote, post_remote, small_max_cells;
    const hbgpu_force_seg *segs;     int32_t nsegs;  /* device */
    double *force_hist;              /* device [max_iters*3*planes*nbody] */
    const hbgpu_peer_msg *sends;     int32_t nsends; /* HOST arrays */
    const hbgpu_peer_msg *recvs;     int32_t nrecvs;
    void *comm;                      /* from hbgpu_comm_init, NULL if 1 rank */
    const void *tmaps;               /* device, from hbgpu_encode_tensor_maps */
    int32_t nblocks, total_tiles, planes, nbody, tile_rows, max_iters;
    int32_t interleaved, tile_pdes;  /* slot layout, tile geometry          */
    double coef[4];
    double D[HBGPU_MAX_TEMPLATED_P * HBGPU_MAX_TEMPLATED_P];
    double ap[HBGPU_MAX_P * HBGPU_NPDE];
} hbgpu_engine_desc;

/* The engine runs on its own non-blocking stream (CUDA graphs cannot be
 * captured on the legacy default stream); every call orders that stream
 * after the caller's `stream` on entry and the caller's stream after it on
 * exit, so the engine behaves as if it ran on `stream`. */
typedef struct hbgpu_engine hbgpu_engine;

int hbgpu_engine_create(const hbgpu_engine_desc *desc, hbgpu_engine **out);
/* priming halo exchange of slot A (driver.py:129) */
int hbgpu_engine_prime(hbgpu_engine *eng, void *stream);
/* `iterations` full iterations: 4 x (stage [+ NCCL + unpack]), norm fold,
 * forces.  use_graph != 0 replays a CUDA graph of one iteration.  The
 * engine counts the iterations it has issued (iterate and step phase 4)
 * and refuses (HBGPU_ERR_ARG, nothing launched) a call that would take the
 * count past desc.max_iters, the capacity of sumsq and force_hist.        */
int hbgpu_engine_iterate(hbgpu_engine *eng, int32_t iterations, int32_t use_graph,
                         void *stream);
/* iterations issued since create / the last rewind */
int hbgpu_engine_iterations_done(const hbgpu_engine *eng);
/* start the history over: issued count = 0, and on `stream` the device
 * iteration counter = 0 and every status key = all-ones (no divergence)  */
int hbgpu_engine_rewind(hbgpu_engine *eng, void *stream);
/* The same schedule split at its exchange points, for a caller that moves
 * the remote halo payloads itself (several ranks' engines in one process):
 * phase -1 = priming halo moves of slot A (local copies + pack), 0..3 = the
 * fused stage kernel of that RK stage (+ norm fold after stage 0), 4 =
 * forces and the iteration counter.  hbgpu_engine_unpack(e, phase) then
 * scatters the receive buffer into the slot that phase wrote.            */
int hbgpu_engine_step(hbgpu_engine *eng, int32_t phase, void *stream);
int hbgpu_engine_unpack(hbgpu_engine *eng, int32_t phase, void *stream);
/* phase 0..3 (a pass phase: single stages, or the paired schedule's 1 and
 * 3) in the two parts the multi-GPU engine overlaps with its exchange:
 * part 0 = the boundary tiles (desc.tile_order[0, nbound_tiles)) and the
 * remote packs -- after it the send buffer is complete; part 1 = the
 * interior tiles, the norm fold (first stage) and the local halo copies.
 * A caller that moves the payloads itself runs part 0, its transfer
 * (concurrently with part 1 if it likes), part 1, then unpack.            */
int hbgpu_engine_step_split(hbgpu_engine *eng, int32_t phase, int32_t part, void *stream);
/* kernels this engine launches per iteration (for launch accounting) */
int hbgpu_engine_launches_per_iteration(const hbgpu_engine *eng);
int hbgpu_engine_destroy(hbgpu_engine *eng);

/* ---- NCCL plumbing (NCCL is dlopen'ed on first use) ---------------------- */
int hbgpu_comm_unique_id(unsigned char id[128]);
int hbgpu_comm_init(const unsigned char id[128], int32_t nranks, int32_t rank,
                    int32_t device, void **comm);
/* all-gather of `count` doubles per rank (ranks stacked in rank order) */
int hbgpu_comm_allgather(void *comm, const double *send, double *recv,
                         int64_t count, void *stream);
int hbgpu_comm_destroy(void *comm);
/* all-reduce of `count` elements: HBGPU_REDUCE_SUM_F64 (doubles, sum) or
 * HBGPU_REDUCE_MIN_U64 (status keys, unsigned min)                        */
#define HBGPU_REDUCE_SUM_F64 0
#define HBGPU_REDUCE_MIN_U64 1
int hbgpu_comm_allreduce(void *comm, const void *send, void *recv, int64_t count,
                         int32_t op, void *stream);
/* one grouped ncclSend / ncclRecv of every listed peer segment (doubles;
 * hbgpu_peer_msg arrays on the HOST) on `stream`: the block-level
 * exchange_halos transport (exchange.py:307-316, one payload per peer)    */
int hbgpu_comm_exchange(void *comm, const double *sendbuf, const hbgpu_peer_msg *sends,
                        int32_t nsends, double *recvbuf, const hbgpu_peer_msg *recvs,
                        int32_t nrecvs, void *stream);
/* HBGPU_OK while the communicator is healthy (or has work in progress);
 * HBGPU_ERR_NCCL with the message when ncclCommGetAsyncError reports an
 * error (a peer failed, a network error).  Poll it while waiting.         */
int hbgpu_comm_async_error(void *comm);
/* ncclCommAbort: frees the communicator and aborts its uncompleted
 * operations, so a rank that failed (or timed out) does not leave its
 * peers blocked in a collective (runtime.py:133-144 aborts the fabric).   */
int hbgpu_comm_abort(void *comm);

/* ---- misc ---------------------------------------------------------------- */
/* sizeof / offsetof of the ABI structs, for binding checks:
 * out[0..5] = sizeof(hbgpu_block, hbgpu_face_target, hbgpu_halo_dir,
 * hbgpu_force_seg, hbgpu_peer_msg, hbgpu_stage_args), out[6] =
 * sizeof(hbgpu_engine_desc), out[7] = offsetof(hbgpu_engine_desc, coef),
 * out[8] = offsetof(hbgpu_stage_args, coef); returns the count written */
int hbgpu_abi_layout(int64_t *out, int32_t n);
int hbgpu_abi_version(void);
const char *hbgpu_last_error(void);
/* kernel launches issued by this library since load (all entry points) */
uint64_t hbgpu_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* HBGPU_H */
