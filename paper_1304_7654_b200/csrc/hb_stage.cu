// hb_stage.cu -- the fused HB Runge-Kutta stage kernel (the hot path).
//
// One launch performs, for every interior cell of every block a rank owns,
// all P snapshots and all 4 pdes of
//
//   R = stencil(q_in) + sum_m D[n][m] q_in[m] + ap[n][p] * sxy      (hbcore.py:184-221)
//   q_out = q_0 - coef * R                                           (hbcore.py:224-245)
//
// plus, fused:
//   * halo forwarding: an interior face cell on a cut is also stored into the
//     paired halo cell of the output slot (local cut) or into the send buffer
//     in the reference's element-major layout (remote cut) -- the
//     _copy_local / _pack of exchange.py:248-261;
//   * divergence keys (hbcore.py:244-245, 279-284);
//   * stage 0: per-(tile, warp) partial sums of R^2 for the residual norm.
//
// Work decomposition.  A tile is one CTA's strip of one block over
// `tile_rows` rows: PT pdes x 256/PT columns (PT = 4: 64 columns of every
// pde; PT = 1: 256 columns of one pde, for blocks at least 192 wide).  Each of
// the 8 consumer warps owns 32 columns of one pde; lane l owns one column and
// marches down the rows keeping rows j-1, j, j+1 of all P snapshots of its
// column in registers (stencil north/south neighbours and the P centres of
// the D-contraction).
//
// Memory pipeline (warp-specialised, TMA).  A ninth warp is the producer: one
// lane streams the tile's rows into shared memory with tensor TMA loads
// (cp.async.bulk.tensor): per row, the stencil box (the strip plus two halo
// columns each side, x PT pdes x P snapshots; split in two boxes when wider
// than TMA's 256-element limit) into a ring of R slots, the strip's q_0 row
// into a ring of Q slots, and the sxy forcing row riding on the stencil
// slot's barrier.  Every slot has a "full" mbarrier (TMA transaction count)
// and an "empty" one the consumer warps arrive on once they stop reading it.
// With ROW_LEAD = 7 every strip starts on a 64-byte DRAM granule: a q_0 row
// costs exactly its bytes and a stencil row one extra granule each side,
// shared with the neighbouring strips (2/32 extra at PT = 1).  CTAs are
// persistent (tiles t = blockIdx.x, +gridDim.x, ...) and the rings stream
// across tile boundaries without draining.
//
// Rounding: every operation is an explicitly rounded DMUL/DADD, in the
// reference's per-point order.  The m == n coupling term (D[n][n] = 0) and
// the zero-amplitude forcing planes contribute signed zeros, reproduced
// exactly by add_signed_zero (hb_common.cuh).

#include "hb_tma.cuh"

#include <cuda.h>
#include <stdlib.h>
#include <string.h>

namespace hbgpu {

// Output rows of the update stages leave by TMA store from the q0 slot they
// replace.  The first stage has no q0 ring; it stages its rows in NOUT own
// slots, so that its store warp forwards the west / east face columns as in
// the other stages and no column-halo pass follows the launch (the engine
// asks hbgpu_stage_first_forwards).  Staging costs the issue-bound first
// stage ~8% at C4's size against plain stores + a 0.23 ms halo pass, but the
// single-stage schedule serves the small cases, where that extra launch is
// 5 of ~60-100 us per iteration (C1, C2).  P > 9 (rings near the shared-
// memory limit) keeps plain stores and the halo pass.
#ifndef HBGPU_FIRST_STAGING
#define HBGPU_FIRST_STAGING 2
#endif
constexpr int first_staging(int P) { return P <= 9 ? HBGPU_FIRST_STAGING : 0; }

template <int P, bool FIRST, int R, int Q, int PT>
struct Smem {
    using G = Geo<PT>;
    static constexpr int BOXD = P * PT * G::BW;                          // doubles per box
    static constexpr int REGION = (BOXD * 8 + 127) / 128 * 128 / 8;      // 128-B aligned
    static constexpr int SXY = G::NSPLIT * REGION;                       // sxy row offset
    static constexpr int SLOT = SXY + G::TCOLS;                          // stencil slot
    static constexpr int QSLOT = P * PT * G::TCOLS;                      // q0 slot
    static constexpr int NQ = FIRST ? 0 : Q;
    // output rows are staged for the TMA store in the q0 slot they replace;
    // the first stage has no q0 ring: first_staging(P) own slots, or plain stores
    static constexpr int NO = FIRST ? first_staging(P) : 0;
    static constexpr int NS = FIRST ? NO : NQ;   // staging slots (either kind)
    static constexpr size_t BAR_OFF = ((size_t)R * SLOT + (size_t)(NQ + NO) * QSLOT) * 8;
    static constexpr size_t BYTES = BAR_OFF + (size_t)(2 * (R + NQ) + NS + NO) * 8;
    static_assert((SLOT * 8) % 128 == 0 && (QSLOT * 8) % 128 == 0, "TMA slots need 128-B alignment");
};

// ---- the pipelined kernel -----------------------------------------------------------

// Resident CTAs per SM the kernel is compiled for: small P needs few
// registers and short rings, and a second CTA per SM halves the rows each
// CTA walks in the small, L2-resident cases (C1: 4 x 256 x 128 cells give a
// CTA ~14 rows of a stage, so its time is the row loop's latency)
#ifndef HBGPU_SMALL_P_CTAS
#define HBGPU_SMALL_P_CTAS 2
#endif
constexpr int stage_ctas_per_sm(int P) { return P <= 5 ? HBGPU_SMALL_P_CTAS : 1; }

template <int P, bool FIRST, int R, int Q, int PT, int MODE>
__global__ void __launch_bounds__(THREADS, stage_ctas_per_sm(P)) stage_tma_kernel(const __grid_constant__ hbgpu_stage_args a) {
    using S = Smem<P, FIRST, R, Q, PT>;
    using G = Geo<PT>;
    static_assert(R >= 3 && Q >= 2, "ring too short");
    extern __shared__ __align__(1024) unsigned char smem[];
    double *ring = reinterpret_cast<double *>(smem);
    double *qring = ring + R * S::SLOT;
    double *oring = qring + S::NQ * S::QSLOT;    // first stage: output staging
    uint64_t *full_in = reinterpret_cast<uint64_t *>(smem + S::BAR_OFF);
    uint64_t *empty_in = full_in + R;
    uint64_t *full_q = empty_in + R;
    uint64_t *empty_q = full_q + S::NQ;          // q0 slot stored out and free
    uint64_t *staged = empty_q + S::NQ;          // output row written to smem
    uint64_t *out_free = staged + S::NS;         // first stage: staging slot free
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int k = 0; k < R; ++k) {
            mbar_init(full_in + k, 1);
            mbar_init(empty_in + k, CW);
        }
        for (int k = 0; k < S::NQ; ++k) {
            mbar_init(full_q + k, 1);
            mbar_init(empty_q + k, 1);
        }
        for (int k = 0; k < S::NS; ++k) mbar_init(staged + k, CW * 32);
        for (int k = 0; k < S::NO; ++k) mbar_init(out_free + k, 1);
        fence_mbar_init();
    }
    __syncthreads();
    const int ntile = tile_end(a);
    const CUtensorMap *maps = reinterpret_cast<const CUtensorMap *>(a.tmaps);
    const bool inter = a.interleaved != 0;

    if (warp == CW) {
        // ------------------------------ producer ------------------------------
        if (lane != 0) return;
        constexpr uint32_t BYTES = S::BOXD * 8 * G::NSPLIT, QBYTES = S::QSLOT * 8, SBYTES = G::TCOLS * 8;
        RingPos pin{0, 0}, pq{0, 0};
        int issued_in = 0, issued_q = 0;   // saturate at the ring size
        for (int k = a.tile_lo + blockIdx.x; k < ntile; k += gridDim.x) {
            const int t = tile_at(a, k);
            const Tile tl = decode_tile<PT>(a, t);
            const CUtensorMap *min = maps + a.in_slot * a.nblocks + tl.bidx;
            const CUtensorMap *mq = maps + 3 * a.nblocks + tl.bidx;   // q0: slot 0, strip box
            const CUtensorMap *ms = maps + 4 * a.nblocks + tl.bidx;   // sxy table
            prefetch_tmap(min);
            const int x = tl.i0 + LEAD - 2;
            // stencil rows; the entry of row r also carries sxy row r-1, the
            // forcing of the row computed while r is the "north" row
            auto put_in = [&](int row, bool with_sxy) {
                if (issued_in >= R) mbar_wait_idle(empty_in + pin.slot, pin.phase ^ 1u);
                else ++issued_in;
                double *dst = ring + pin.slot * S::SLOT;
                mbar_expect_tx(full_in + pin.slot, with_sxy ? BYTES + SBYTES : BYTES);
#pragma unroll
                for (int k = 0; k < G::NSPLIT; ++k)
                    load_rows<PT>(dst + k * S::REGION, min, x + k * (G::TCOLS / G::NSPLIT), tl.pde0, row, inter,
                                  full_in + pin.slot);
                if (with_sxy) tma_load_2d(dst + S::SXY, ms, tl.i0 - 1, row - 2, full_in + pin.slot);
                pin = advance<R>(pin);
            };
            put_in(tl.j0 - 1, false);
            put_in(tl.j0, false);
            for (int j = tl.j0; j <= tl.j1; ++j) {
                put_in(j + 1, true);
                if (!FIRST) {
                    if (issued_q >= Q) mbar_wait_idle(empty_q + pq.slot, pq.phase ^ 1u);
                    else ++issued_q;
                    mbar_expect_tx(full_q + pq.slot, QBYTES);
                    load_rows<PT>(qring + pq.slot * S::QSLOT, mq, x + 2, tl.pde0, j, inter, full_q + pq.slot);
                    pq = advance<Q>(pq);
                }
            }
        }
        return;
    }
    constexpr bool TSTORE = !FIRST || S::NO > 0;   // rows leave by TMA store
    if (warp == CW + 1) {
        if (!TSTORE) return;
        // ------------------------------ store warp ------------------------------
        // one TMA store per output row once all consumer threads have staged
        // it; the staging slot is handed back (to the q0 loads, or to the
        // consumers in the first stage) when the store has read it
        // The warp also forwards the strip's west / east face columns, cells
        // i = 1 and i = ni, read back from the staged row: one lane per
        // (plane, pde) value, off the consumers' critical path.
        RingPos ps{0, 0};
        for (int k = a.tile_lo + blockIdx.x; k < ntile; k += gridDim.x) {
            const int t = tile_at(a, k);
            const Tile tl = decode_tile<PT>(a, t);
            const CUtensorMap *mo = maps + (5 + a.out_slot) * a.nblocks + tl.bidx;
            if (lane == 0) prefetch_tmap(mo);
            const hbgpu_block b = a.blocks[tl.bidx];
            const int64_t west = tl.i0 == 1 ? b.face_off[2] : -1;
            const int64_t east = tl.i0 + G::TCOLS > b.ni ? b.face_off[3] : -1;
            constexpr int KV = (P * PT + 31) / 32;   // column values per lane
            const int col_e = b.ni - tl.i0;
            // targets are loaded a row ahead; values are read from the staged
            // row into registers before the slot is handed back
            FaceHit tw = load_target(a.faces, west, tl.j0 - 1), te = load_target(a.faces, east, tl.j0 - 1);
            for (int j = tl.j0; j <= tl.j1; ++j) {
                mbar_wait(staged + ps.slot, ps.phase);
                const double *src = FIRST ? oring + ps.slot * S::QSLOT : qring + ps.slot * S::QSLOT;
                if (lane == 0) {
                    store_rows(mo, src, tl.i0 + LEAD, tl.pde0, j, inter);
                    bulk_commit();
                }
                double vw[KV], ve[KV];
#pragma unroll
                for (int c = 0; c < KV; ++c) {   // value k = n * PT + pde within the tile
                    const int k = lane + 32 * c;
                    if (k < P * PT) {
                        if (tw.ps != 0) vw[c] = src[k * G::TCOLS];
                        if (te.ps != 0) ve[c] = src[k * G::TCOLS + col_e];
                    }
                }
                const bool more = j < tl.j1;
                const FaceHit nw = load_target(a.faces, more ? west : -1, j),
                              ne = load_target(a.faces, more ? east : -1, j);
                __syncwarp();
                if (lane == 0) {
                    bulk_wait_read_all();
                    mbar_arrive(FIRST ? out_free + ps.slot : empty_q + ps.slot);
                }
#pragma unroll
                for (int c = 0; c < KV; ++c) {
                    const int k = lane + 32 * c;
                    if (k < P * PT) {
                        const int n = k / PT, pp = k - n * PT;
                        if (tw.ps != 0) forward(tw, a.out, a.sendbuf, n, tl.pde0 + pp, vw[c]);
                        if (te.ps != 0) forward(te, a.out, a.sendbuf, n, tl.pde0 + pp, ve[c]);
                    }
                }
                tw = nw;
                te = ne;
                ps = advance<S::NS>(ps);
            }
        }
        if (lane == 0) bulk_wait_all();
        return;
    }

    // -------------------------------- consumers ---------------------------------
    const int pp = warp % PT;                     // pde within the tile
    const int cw = warp / PT;                     // column warp within the strip
    const int col0 = 32 * cw + lane;              // this lane's column within the strip
    // offset of this lane's column (+2 halo columns) inside a stencil slot
    const int in_off = (cw / G::CWPR) * S::REGION + pp * G::BW + 32 * (cw % G::CWPR) + lane + 2;
    const int q_off = pp * G::TCOLS + col0;
    const int gstage = (*a.iter) * 4 + a.stage + 1;
    const double coef = a.coef;
    RingPos cin{0, 0}, cq{0, 0}, co{0, 0};
    int used_out = 0;   // first stage: staging slots handed out so far (saturates)
    int ap_pde = -1;
    double ap[P];
    double dk[P / 2 + 1];   // dk[k] = D[m+k][m] for every m (circulant)
#pragma unroll
    for (int k = 1; k <= P / 2; ++k) dk[k] = a.D[k * P];
    for (int k = a.tile_lo + blockIdx.x; k < ntile; k += gridDim.x) {
            const int t = tile_at(a, k);
        const Tile tl = decode_tile<PT>(a, t);
        const int p = tl.pde0 + pp;
        if (p != ap_pde) {
#pragma unroll
            for (int n = 0; n < P; ++n) ap[n] = a.ap[n * NPDE + p];
            ap_pde = p;
        }
        // by value: the output stores must not force re-reads of the descriptor
        const hbgpu_block b = a.blocks[tl.bidx];
        const int ni = b.ni, nj = b.nj;
        const double nu_h2 = b.nu_h2, adv_2h = b.adv_2h;
        const int i = tl.i0 + col0;
        const bool live = i <= ni;
        // plain stores: columns past the TMA store extent, or every column
        const bool tail = live && (!TSTORE || i > store_cols(ni));
        double *const tail_out = a.out + b.base + (int64_t)p * b.ps + LEAD + i;
        const int64_t ps4 = b.ps * NPDE;

        // south / north face rows are forwarded here; west / east columns by
        // the store warp (update stages) or the engine's post pass (stage 1)
        FaceHit trow = row_target(a.faces, b, i, tl.j0, live);

        // rows j0-1 and j0 -> registers; release row j0-1
        // rows j-1, j, j+1 of this lane's column, rotated by the row step's
        // argument order (the loop below is unrolled by 3: no register moves)
        double ra[P], rb[P], rc3[P];
        {
            const RingPos c1 = advance<R>(cin);
            mbar_wait(full_in + cin.slot, cin.phase);
            mbar_wait(full_in + c1.slot, c1.phase);
            const double *r0 = ring + cin.slot * S::SLOT + in_off;
            const double *r1 = ring + c1.slot * S::SLOT + in_off;
#pragma unroll
            for (int m = 0; m < P; ++m) {
                ra[m] = r0[m * PT * G::BW];
                rb[m] = r1[m * PT * G::BW];
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(empty_in + cin.slot);
            cin = c1;   // entry of the current row j
        }
        double nrm = 0.0;

        auto row_step = [&](const int j, double(&up)[P], double(&cur)[P], double(&dn)[P]) {
            // prefetch the next row's halo targets (boundary cells only)
            const FaceHit nrow = row_target(a.faces, b, i, j + 1, live && j < tl.j1);

            const RingPos nx = advance<R>(cin);
            mbar_wait(full_in + nx.slot, nx.phase);
            const double *rc = ring + cin.slot * S::SLOT + in_off;
            const double *rn = ring + nx.slot * S::SLOT + in_off;
            const double sv = ring[nx.slot * S::SLOT + S::SXY + col0];   // sxy of row j
#pragma unroll
            for (int m = 0; m < P; ++m) dn[m] = rn[m * PT * G::BW];
            const double *qv = nullptr;
            if (!FIRST) {
                mbar_wait(full_q + cq.slot, cq.phase);
                qv = qring + cq.slot * S::QSLOT + q_off;
            }

            // All P outputs in lockstep, branch-free: each step below is P
            // independent rounded operations (one per snapshot), so the P
            // dependency chains overlap.  Per point the rounding sequence is
            // the reference's: stencil, then m ascending, then forcing
            // (hbcore.py:193-221 is this same pass structure).
            double v[P], o[P];
            {
                double w[P], e[P];
#pragma unroll
                for (int n = 0; n < P; ++n) {
                    w[n] = rc[n * PT * G::BW - 1];
                    e[n] = rc[n * PT * G::BW + 1];
                }
#pragma unroll
                for (int n = 0; n < P; ++n) o[n] = rmul(4.0, cur[n]);
#pragma unroll
                for (int n = 0; n < P; ++n) o[n] = rsub(o[n], w[n]);
#pragma unroll
                for (int n = 0; n < P; ++n) o[n] = rsub(o[n], e[n]);
#pragma unroll
                for (int n = 0; n < P; ++n) o[n] = rsub(o[n], up[n]);
#pragma unroll
                for (int n = 0; n < P; ++n) o[n] = rsub(o[n], dn[n]);
#pragma unroll
                for (int n = 0; n < P; ++n) o[n] = rmul(o[n], nu_h2);
#pragma unroll
                for (int n = 0; n < P; ++n) o[n] = radd(o[n], rmul(rsub(e[n], w[n]), adv_2h));
            }
            // D is the spectral matrix: circulant and exactly antisymmetric
            // (D[m+k][m] == dk[k] == -D[m-k][m] bit for bit, checked on the
            // host), so column m's product for row m+k is, negated, row
            // m-k's: one DMUL feeds a DADD and a DSUB with the reference's
            // rounding (x + (-y) == x - y, (-d) y == -(d y)).  The D[m][m]
            // == +0 term and the zero-amplitude forcing planes add 0*x, a
            // signed zero formed on the integer pipe (zero_times).
#pragma unroll
            for (int m = 0; m < P; ++m) {
                o[m] = radd(o[m], zero_times(cur[m]));
#pragma unroll
                for (int k = 1; k <= P / 2; ++k) {
                    const double prod = rmul(dk[k], cur[m]);
                    o[(m + k) % P] = radd(o[(m + k) % P], prod);
                    o[(m + P - k) % P] = rsub(o[(m + P - k) % P], prod);
                }
            }
            const double sv0 = zero_times(sv);
#pragma unroll
            for (int n = 0; n < P; ++n) {
                o[n] = radd(o[n], forced_plane(n) ? rmul(ap[n], sv) : sv0);
                const double base = FIRST ? cur[n] : qv[n * PT * G::TCOLS];
                v[n] = rsub(base, rmul(coef, o[n]));
                if (MODE == 1) v[n] = base;   // measurement variant: same traffic, no arithmetic
            }
            if (FIRST && live) {
                // the residual norm is not a reference quantity (no bitwise
                // contract; tolerance 1e-12 vs an exactly rounded sum), so it
                // may use fused multiply-adds
#pragma unroll
                for (int n = 0; n < P; ++n) nrm = __fma_rn(o[n], o[n], nrm);
            }

            if (TSTORE) {
                // stage the output row for the TMA store: in place of the q0
                // row it replaces, or (first stage) in an output staging slot
                double *stage_row;
                if (FIRST) {
                    if (used_out >= S::NO) mbar_wait(out_free + co.slot, co.phase ^ 1u);
                    else ++used_out;
                    stage_row = oring + co.slot * S::QSLOT + q_off;
                } else {
                    stage_row = qring + cq.slot * S::QSLOT + q_off;
                }
#pragma unroll
                for (int n = 0; n < P; ++n) stage_row[n * PT * G::TCOLS] = v[n];
                fence_proxy_async_smem();
                mbar_arrive(staged + (FIRST ? co.slot : cq.slot));
                if (FIRST) co = advance<S::NO>(co);
            }
            const int64_t row = (int64_t)j * b.rs;
            if (tail) {
#pragma unroll
                for (int n = 0; n < P; ++n) tail_out[n * ps4 + row] = v[n];
            }
            if (trow.ps != 0) {
#pragma unroll
                for (int n = 0; n < P; ++n) forward(trow, a.out, a.sendbuf, n, p, v[n]);
            }
            bool ok = true;
#pragma unroll
            for (int n = 0; n < P; ++n) ok = ok && (MODE == 1 || finite_fp(v[n]));
            const bool bad = !ok;
            if (bad && live) {
                for (int n = 0; n < P; ++n)
                    if (nonfinite(v[n])) {
                        long long lin = (((long long)(n * NPDE + p) * nj + (j - 1)) * ni) + (i - 1);
                        atomicMin(a.status + tl.bidx, divergence_key(gstage, lin));
                    }
            }
            trow = nrow;
            __syncwarp();
            if (lane == 0) mbar_arrive(empty_in + cin.slot);   // row j no longer read
            cin = nx;
            if (!FIRST) cq = advance<Q>(cq);
        };
        int j = tl.j0;
        for (; j + 2 <= tl.j1; j += 3) {
            row_step(j, ra, rb, rc3);
            row_step(j + 1, rb, rc3, ra);
            row_step(j + 2, rc3, ra, rb);
        }
        if (j <= tl.j1) {
            row_step(j, ra, rb, rc3);
            if (j + 1 <= tl.j1) row_step(j + 1, rb, rc3, ra);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(empty_in + cin.slot);   // row j1+1
        cin = advance<R>(cin);
        if (FIRST && a.norm_part != nullptr) {
            const double s = warp_sum(nrm);
            if (lane == 0) a.norm_part[(int64_t)t * CW + warp] = s;
        }
    }
}

// ---- generic snapshot count (P > HBGPU_MAX_TEMPLATED_P) --------------------------
// One CTA of CW warps (same warp -> (pde, columns) map) per tile, operands
// through L1, D from shared memory.  Same arithmetic sequence; used for e.g.
// the 63-plane tc1-full catalog case.
template <int PT>
__global__ void __launch_bounds__(CW * 32) stage_kernel_generic(const __grid_constant__ hbgpu_stage_args a) {
    extern __shared__ double sh[];
    const int P = a.planes;
    for (int k = threadIdx.x; k < P * P; k += blockDim.x) sh[k] = a.dmat[k];
    __syncthreads();
    const double *D = sh;
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int t = tile_at(a, a.tile_lo + blockIdx.x);
    const Tile tl = decode_tile<PT>(a, t);
    const int p = tl.pde0 + warp % PT;
    const hbgpu_block &b = a.blocks[tl.bidx];
    const int ni = b.ni, nj = b.nj;
    const int64_t rstride = b.rs;
    const int64_t ps4 = b.ps * NPDE;
    const int i = tl.i0 + 32 * (warp / PT) + lane;
    const bool live = i <= ni;
    const bool first = a.stage == 0;
    const int gstage = (*a.iter) * 4 + a.stage + 1;
    double nrm = 0.0;
    if (live) {
        const int64_t col = b.base + (int64_t)b.ps * p + LEAD + i;
        const double *in = a.in + col;
        for (int j = tl.j0; j <= tl.j1; ++j) {
            const int64_t row = (int64_t)j * rstride;
            const double sv = a.sxy[b.sxy_off + (int64_t)(j - 1) * b.sxy_pitch + (i - 1)];
            FaceHit trow, tcol;
            cell_targets(a.faces, b, i, j, true, trow, tcol);
            for (int n = 0; n < P; ++n) {
                const double *c = in + n * ps4 + row;
                double o = stencil(c[0], c[-1], c[1], c[-rstride], c[rstride], b.nu_h2, b.adv_2h);
                for (int m = 0; m < P; ++m) o = radd(o, rmul(D[n * P + m], in[m * ps4 + row]));
                o = radd(o, rmul(a.ap[n * NPDE + p], sv));
                const double base = first ? c[0] : a.q0[col + n * ps4 + row];
                const double v = rsub(base, rmul(a.coef, o));
                a.out[col + n * ps4 + row] = v;
                if (first) nrm = radd(nrm, rmul(o, o));
                forward(trow, a.out, a.sendbuf, n, p, v);
                forward(tcol, a.out, a.sendbuf, n, p, v);
                if (nonfinite(v)) {
                    long long lin = (((long long)(n * NPDE + p) * nj + (j - 1)) * ni) + (i - 1);
                    atomicMin(a.status + tl.bidx, divergence_key(gstage, lin));
                }
            }
        }
    }
    if (first && a.norm_part != nullptr) {
        const double s = warp_sum(nrm);
        if (lane == 0) a.norm_part[(int64_t)t * CW + warp] = s;
    }
}

// ---- launch -------------------------------------------------------------------

int current_device() {
    int dev = -1;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= HB_MAX_DEVICES) {
        hbgpu_set_error("hbgpu: current device %d unusable (limit %d devices)", dev, HB_MAX_DEVICES);
        return -1;
    }
    return dev;
}

int persistent_grid(int resident, int tiles) {
    int grid = min(resident, tiles);
    if (const char *cap = getenv("HBGPU_GRID_LIMIT")) {
        const int c = atoi(cap);
        if (c > 0) grid = min(grid, c);
    }
    return max(grid, 1);
}

struct Launch {
    void (*fn)(hbgpu_stage_args) = nullptr;
    size_t smem = 0;
    int grid = 0;   // persistent CTAs: SMs x resident CTAs per SM
    bool ready = false;
};

template <int P, bool FIRST, int R, int Q, int PT, int MODE>
static int prepare(Launch &L) {
    if (L.ready) return HBGPU_OK;
    L.fn = stage_tma_kernel<P, FIRST, R, Q, PT, MODE>;
    L.smem = Smem<P, FIRST, R, Q, PT>::BYTES;
    if (cudaFuncSetAttribute(L.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.smem) != cudaSuccess)
        return hbgpu_check_launch("stage kernel smem attribute");
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, L.fn, THREADS, L.smem) != cudaSuccess ||
        per_sm < 1)
        return hbgpu_check_launch("stage kernel occupancy");
    L.grid = sms * per_sm;
    L.ready = true;
    return HBGPU_OK;
}

// Ring depths per snapshot count: R stencil rows for the update stages, RF
// for the first stage (no q0 ring, so its rows go deeper), Q q0 rows.  One
// CTA (8 consumer warps) per SM; the smem budget is ~227 KB.
#ifndef HBGPU_DEPTH_R   // measurement builds may override the default depths
#define HBGPU_DEPTH_R 4
#endif
#ifndef HBGPU_DEPTH_RF
#define HBGPU_DEPTH_RF 7
#endif
#ifndef HBGPU_DEPTH_Q
#define HBGPU_DEPTH_Q 3
#endif
template <int P> struct Depth {
    static constexpr int R = HBGPU_DEPTH_R, RF = HBGPU_DEPTH_RF, Q = HBGPU_DEPTH_Q;
};
#if HBGPU_SMALL_P_CTAS == 2   // two CTAs per SM: at most ~113 KB each
template <> struct Depth<1> { static constexpr int R = 6, RF = 8, Q = 4; };
template <> struct Depth<3> { static constexpr int R = 5, RF = 8, Q = 4; };
template <> struct Depth<5> { static constexpr int R = 4, RF = 6, Q = 3; };
#else
template <> struct Depth<1> { static constexpr int R = 8, RF = 12, Q = 6; };
template <> struct Depth<3> { static constexpr int R = 8, RF = 12, Q = 6; };
template <> struct Depth<5> { static constexpr int R = 6, RF = 10, Q = 5; };
#endif
template <> struct Depth<13> { static constexpr int R = 4, RF = 6, Q = 2; };
template <> struct Depth<15> { static constexpr int R = 4, RF = 5, Q = 2; };
template <> struct Depth<17> { static constexpr int R = 4, RF = 5, Q = 2; };

template <int P, int PT, int MODE>
static int launch_cfg(const hbgpu_stage_args &a, cudaStream_t s, bool prepare_only) {
    using D = Depth<P>;
    // the smem attribute and the occupancy grid are per device
    static Launch first_d[HB_MAX_DEVICES], rest_d[HB_MAX_DEVICES];
    const int dev = current_device();
    if (dev < 0) return HBGPU_ERR_CUDA;
    Launch &first = first_d[dev], &rest = rest_d[dev];
    int rc = prepare<P, true, D::RF, D::Q, PT, MODE>(first);
    if (!rc) rc = prepare<P, false, D::R, D::Q, PT, MODE>(rest);
    if (rc || prepare_only) return rc;
    if (a.tmaps == nullptr) {
        hbgpu_set_error("hbgpu_stage: args->tmaps is required (hbgpu_encode_tensor_maps)");
        return HBGPU_ERR_ARG;
    }
    Launch &L = a.stage == 0 ? first : rest;
    const int grid = persistent_grid(L.grid, tile_end(a) - a.tile_lo);
    L.fn<<<grid, THREADS, L.smem, s>>>(a);
    hbgpu_count_launch(1);
    return hbgpu_check_launch("hbgpu_stage");
}

template <int P>
static int launch_p(const hbgpu_stage_args &a, cudaStream_t s, bool prepare_only) {
#ifdef HBGPU_MEASURE_NOMATH
    // measurement builds only (-DHBGPU_MEASURE_NOMATH, never the shipped
    // library): P = 9 with the arithmetic replaced by a copy of q0, the
    // same pipeline and traffic
    if constexpr (P == 9)
        return a.tile_pdes == 1 ? launch_cfg<P, 1, 1>(a, s, prepare_only) : launch_cfg<P, 4, 1>(a, s, prepare_only);
#endif
    return a.tile_pdes == 1 ? launch_cfg<P, 1, 0>(a, s, prepare_only) : launch_cfg<P, 4, 0>(a, s, prepare_only);
}

// The templated kernel multiplies by dk[k] = D[k][0] for every D[m+k][m] and
// shares each product between rows m+k and m-k; that is exact only for the
// spectral matrix's bitwise circulant, antisymmetric structure (hbcore.py:
// 88-94 computes D from the wrapped d = n - m in [-N_H, N_H] alone, and
// D(-d) = -D(d) exactly).
static bool circulant_antisymmetric(const double *D, int P) {
    for (int m = 0; m < P; ++m) {
        uint64_t diag;
        memcpy(&diag, D + m * P + m, 8);
        if (diag != 0) return false;
        for (int k = 1; k <= P / 2; ++k) {
            uint64_t x, y, d0;
            memcpy(&x, D + ((m + k) % P) * P + m, 8);
            memcpy(&y, D + ((m + P - k) % P) * P + m, 8);
            memcpy(&d0, D + k * P, 8);
            if (x != d0 || x != (y ^ 0x8000000000000000ull)) return false;
        }
    }
    return true;
}

static int dispatch(const hbgpu_stage_args &a, cudaStream_t s, bool prepare_only) {
    if (a.tile_pdes != 1 && a.tile_pdes != 4) {
        hbgpu_set_error("hbgpu_stage: tile_pdes must be 1 or 4, got %d", a.tile_pdes);
        return HBGPU_ERR_ARG;
    }
    if (a.pair != 0) {
        if (!prepare_only && !circulant_antisymmetric(a.D, a.planes)) {
            hbgpu_set_error("hbgpu_stage: D must be the spectral matrix (+0.0 diagonal, D[m+k][m] == D[k][0] == -D[m-k][m])");
            return HBGPU_ERR_ARG;
        }
        return pair_dispatch(a, s, prepare_only);
    }
    if (!prepare_only && a.planes <= HBGPU_MAX_TEMPLATED_P && !circulant_antisymmetric(a.D, a.planes)) {
        hbgpu_set_error("hbgpu_stage: D must be the spectral matrix (+0.0 diagonal, D[m+k][m] == D[k][0] == -D[m-k][m])");
        return HBGPU_ERR_ARG;
    }
    switch (a.planes) {
        case 1: return launch_p<1>(a, s, prepare_only);
        case 3: return launch_p<3>(a, s, prepare_only);
        case 5: return launch_p<5>(a, s, prepare_only);
        case 7: return launch_p<7>(a, s, prepare_only);
        case 9: return launch_p<9>(a, s, prepare_only);
        case 11: return launch_p<11>(a, s, prepare_only);
        case 13: return launch_p<13>(a, s, prepare_only);
        case 15: return launch_p<15>(a, s, prepare_only);
        case 17: return launch_p<17>(a, s, prepare_only);
        default: break;
    }
    auto kern = a.tile_pdes == 1 ? stage_kernel_generic<1> : stage_kernel_generic<4>;
    const size_t sm = sizeof(double) * (size_t)a.planes * a.planes;
    if (sm > 48 * 1024 && cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm) !=
                              cudaSuccess)
        return hbgpu_check_launch("generic stage smem attribute");
    if (prepare_only) return HBGPU_OK;
    if (a.dmat == nullptr) {
        hbgpu_set_error("hbgpu_stage: P=%d needs args->dmat", a.planes);
        return HBGPU_ERR_ARG;
    }
    if (tile_end(a) <= a.tile_lo) return HBGPU_OK;
    kern<<<tile_end(a) - a.tile_lo, CW * 32, sm, s>>>(a);
    hbgpu_count_launch(1);
    return hbgpu_check_launch("hbgpu_stage");
}

// ---- tensor maps ------------------------------------------------------------------

typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *,
                                  CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                  CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    if (fn == nullptr) {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    }
    return fn;
}

}  // namespace hbgpu

// Function attributes and occupancy are resolved once per kernel instantiation,
// before any stream capture (the engine calls this at creation).
extern "C" int hbgpu_stage_prepare(int32_t planes) {
    hbgpu_stage_args a;
    memset(&a, 0, sizeof(a));
    a.planes = planes;
    int rc = HBGPU_OK;
    for (int pt : {1, 4}) {
        a.tile_pdes = pt;
        a.pair = 0;
        rc = rc ? rc : hbgpu::dispatch(a, nullptr, true);
        if (planes <= HBGPU_MAX_PAIR_P) {
            a.pair = 1;
            rc = rc ? rc : hbgpu::dispatch(a, nullptr, true);
        }
    }
    return rc;
}

extern "C" int hbgpu_stage_first_forwards(int32_t planes) {
    // the templated TMA kernels (odd P) with first-stage staging slots
    return planes >= 1 && planes <= 9 && (planes & 1) && hbgpu::first_staging(planes) > 0 ? 1 : 0;
}

extern "C" int hbgpu_stage(const hbgpu_stage_args *args, void *stream) {
    if (args == nullptr || args->total_tiles <= 0 || args->planes < 1 || args->planes > HBGPU_MAX_P ||
        args->in_slot < 0 || args->in_slot > 2) {
        hbgpu_set_error("hbgpu_stage: bad arguments");
        return HBGPU_ERR_ARG;
    }
    const int end = hbgpu::tile_end(*args);
    if (args->tile_lo < 0 || end > args->total_tiles || args->tile_lo > end) {
        hbgpu_set_error("hbgpu_stage: tile range [%d, %d) outside [0, %d)", args->tile_lo, end, args->total_tiles);
        return HBGPU_ERR_ARG;
    }
    if (end == args->tile_lo) return HBGPU_OK;   // an empty part of a split stage
    return hbgpu::dispatch(*args, (cudaStream_t)stream, false);
}

extern "C" int hbgpu_encode_tensor_maps(double *const slot[3], const double *sxy, const hbgpu_block *blocks,
                                        int32_t nblocks, int32_t planes, int32_t tile_pdes, void *out_host,
                                        int64_t out_bytes) {
    using namespace hbgpu;
    if ((int64_t)sizeof(CUtensorMap) * HBGPU_TMAP_SETS * nblocks > out_bytes || planes < 1 || planes > 256 ||
        (tile_pdes != 1 && tile_pdes != 4)) {
        hbgpu_set_error("hbgpu_encode_tensor_maps: output too small, bad planes or tile_pdes");
        return HBGPU_ERR_ARG;
    }
    EncodeTiledFn fn = encode_fn();
    if (fn == nullptr) {
        hbgpu_set_error("cuTensorMapEncodeTiled unavailable from the driver");
        return HBGPU_ERR_CUDA;
    }
    // L2 sector promotion of the TMA fetches; HBGPU_L2_PROMOTION = 0, 64, 128
    // or 256 overrides (measurements: 64 B best on C4)
    CUtensorMapL2promotion promo = CU_TENSOR_MAP_L2_PROMOTION_L2_64B;
    if (const char *env = getenv("HBGPU_L2_PROMOTION")) {
        const int v = atoi(env);
        promo = v == 64 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
              : v == 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
              : v == 256 ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B : CU_TENSOR_MAP_L2_PROMOTION_NONE;
    }
    const cuuint32_t tcols = (cuuint32_t)(256 / tile_pdes);
    const cuuint32_t bw = tile_pdes == 1 ? Geo<1>::BW : Geo<4>::BW;
    CUtensorMap *maps = reinterpret_cast<CUtensorMap *>(out_host);
    // sets 0..2: stencil boxes over slots 0..2; set 3: q0 box over slot 0;
    // set 4: 2-D sxy table box (strip columns x 1 row); sets 5..7: store
    // boxes over slots 0..2, column extent clipped after cell ni
    for (int s = 0; s < HBGPU_TMAP_SETS; ++s) {
        for (int k = 0; k < nblocks; ++k) {
            const hbgpu_block &b = blocks[k];
            CUresult r;
            if (s != 4) {
                // dimension order follows the layout so the strides nest:
                // plane-major (cols, rows, pde, plane), interleaved (cols, pde,
                // plane, rows); both land in smem as [plane][pde][cols]
                const bool inter = b.rs > b.ps;
                // sets 8 / 9: strip-wide row box / one 8-column granule over the
                // band slot (slot 2), read by the paired-stage kernel
                const cuuint32_t w = s < 3 ? bw : s == 9 ? 8u : tcols;
                const cuuint32_t npd = (cuuint32_t)tile_pdes;
                // store extent: columns up to store_cols(ni), a 64-B boundary,
                // so no store granule reaches the east halo cell (the kernel
                // writes the <= 7 columns past it with plain stores)
                const cuuint64_t cols = (s >= 5 && s <= 7) ? (cuuint64_t)(LEAD + 1 + store_cols(b.ni)) : (cuuint64_t)b.pitch;
                const int slot_k = s < 3 ? s : s == 3 ? 0 : s <= 7 ? s - 5 : 2;
                cuuint64_t dims[4], strides[3];
                cuuint32_t box[4];
                if (inter) {
                    cuuint64_t d[4] = {cols, (cuuint64_t)NPDE, (cuuint64_t)planes,
                                       (cuuint64_t)(b.nj + 2)};
                    cuuint64_t st[3] = {(cuuint64_t)b.ps * 8, (cuuint64_t)b.ps * 8 * NPDE, (cuuint64_t)b.rs * 8};
                    cuuint32_t bx[4] = {w, npd, (cuuint32_t)planes, 1};
                    memcpy(dims, d, sizeof(d));
                    memcpy(strides, st, sizeof(st));
                    memcpy(box, bx, sizeof(bx));
                } else {
                    cuuint64_t d[4] = {cols, (cuuint64_t)(b.nj + 2), (cuuint64_t)NPDE,
                                       (cuuint64_t)planes};
                    cuuint64_t st[3] = {(cuuint64_t)b.rs * 8, (cuuint64_t)b.ps * 8, (cuuint64_t)b.ps * 8 * NPDE};
                    cuuint32_t bx[4] = {w, 1, npd, (cuuint32_t)planes};
                    memcpy(dims, d, sizeof(d));
                    memcpy(strides, st, sizeof(st));
                    memcpy(box, bx, sizeof(bx));
                }
                cuuint32_t estr[4] = {1, 1, 1, 1};
                r = fn(&maps[s * nblocks + k], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4,
                       (void *)(slot[slot_k] + b.base), dims, strides, box, estr,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, promo,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            } else {
                cuuint64_t dims[2] = {(cuuint64_t)b.ni, (cuuint64_t)b.nj};
                cuuint64_t strides[1] = {(cuuint64_t)b.sxy_pitch * 8};
                cuuint32_t box[2] = {tcols, 1};
                cuuint32_t estr[2] = {1, 1};
                r = fn(&maps[s * nblocks + k], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2,
                       (void *)(sxy + b.sxy_off), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                       CU_TENSOR_MAP_SWIZZLE_NONE, promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            }
            if (r != CUDA_SUCCESS) {
                hbgpu_set_error("cuTensorMapEncodeTiled failed (%d) for set %d block %d", (int)r, s, k);
                return HBGPU_ERR_CUDA;
            }
        }
    }
    return HBGPU_OK;
}
