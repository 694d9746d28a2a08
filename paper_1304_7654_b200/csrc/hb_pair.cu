// hb_pair.cu -- two RK stages per pass.
//
// Stages 2-4 of the single-stage kernel are HBM-bound (they read q_{s-1} and
// q_0 and write q_s: 96 B per unit) while their arithmetic would fit in far
// less time.  Pairing stages (0, 1) and (2, 3) halves the traffic: a tile
// computes the first stage's values v1 row by row and, one row behind, the
// second stage's v2 from them, without v1 ever going to HBM.
//
// The catch is the stencil at the tile's edges: v2 at the first / last
// column and row of a tile needs v1 just outside it -- in the neighbouring
// strip or row tile (another CTA) or across a block face.  Those values come
// from the band slot (slot 2): before each pair, hbgpu_band computes the
// first stage at every tile-perimeter cell (about 1.6% of the cells at C4),
// stores it there at the cell itself, and forwards cut-face cells into the
// band slot's halo ring (and the send buffer for remote cuts).  Every value
// is computed with the reference's per-point rounding wherever it is
// computed, so the redundant copies are bitwise the tile's own.
//
//   iteration:  band(0)  pair(0,1) -> slot 1   band(2)  pair(2,3) -> slot 0
//               (+ halo exchange after each, a full halo pass after the last)
//
// hbgpu_band (this file) is a plain kernel: one thread per (perimeter cell,
// pde) computing all P snapshots.

#include "hb_tma.cuh"

#include <stdlib.h>
#include <string.h>

namespace hbgpu {

// ---- band: the first stage of a pair at the tile-perimeter cells -----------------

// Segment kinds: dir 0 = a row run (threads along i), dir 1 = a column run
// (threads along j), dir 2 = two adjacent columns i, i+1 (both face columns
// of a block 2 cells wide): a 128-thread block takes 64 rows of both, so the
// two columns' overlapping stencil sectors are fetched once into L1.
template <int P>
__global__ void __launch_bounds__(128) band_kernel(const __grid_constant__ hbgpu_stage_args a) {
    const hbgpu_band_seg sg = a.band_segs[blockIdx.y];
    int e, di = 0;
    if (sg.dir == 2) {
        e = blockIdx.x * 64 + (threadIdx.x & 63);
        di = threadIdx.x >> 6;
    } else {
        e = blockIdx.x * blockDim.x + threadIdx.x;
    }
    if (e >= sg.len) return;
    const int p = blockIdx.z;
    const hbgpu_block b = a.blocks[sg.block];
    const int j = sg.j + (sg.dir ? e : 0);
    const int i = sg.i + (sg.dir ? di : e);
    // column runs skip the band rows (the row runs own those cells)
    const bool column = sg.dir != 0;
    if (column && ((j - 1) % a.tile_rows == 0 || j % a.tile_rows == 0 || j == b.nj)) return;
    // A single face column's cell is then stored as a whole 32-byte sector
    // (no partial-sector fill in L2) when the rest of its sector holds no
    // value anyone reads: cell 1's sector is cells 1..4 (LEAD + 1 = 8), cell
    // ni's is cells ni-3..ni when ni % 4 == 0 -- not the east halo cell ni+1,
    // which a neighbour forwards into -- and with ni >= 8 neither holds the
    // other face column.  Otherwise (and for two-column runs) plain stores.
    const bool sector_store = sg.dir == 1 && b.ni % 4 == 0 && b.ni >= 8;
    const int64_t ps4 = b.ps * NPDE;
    const int64_t cell = b.base + (int64_t)p * b.ps + (int64_t)j * b.rs + LEAD + i;
    const double *c = a.in + cell;
    const bool first = a.stage == 0;
    const double sv = a.sxy[b.sxy_off + (int64_t)(j - 1) * b.sxy_pitch + (i - 1)];
    // every load first (5-6 P independent loads in flight), then the arithmetic
    double cur[P], wv[P], ev[P], sv_[P], nv[P], bq[P];
#pragma unroll
    for (int m = 0; m < P; ++m) {
        const double *cm = c + m * ps4;
        cur[m] = __ldg(cm);
        wv[m] = __ldg(cm - 1);
        ev[m] = __ldg(cm + 1);
        sv_[m] = __ldg(cm - b.rs);
        nv[m] = __ldg(cm + b.rs);
        bq[m] = first ? cur[m] : __ldg(a.q0 + cell + m * ps4);
    }
    FaceHit trow{0, 0}, tcol{0, 0};
    if (j == 1) trow = load_target(a.faces, b.face_off[0], i - 1);
    else if (j == b.nj) trow = load_target(a.faces, b.face_off[1], i - 1);
    if (i == 1) tcol = load_target(a.faces, b.face_off[2], j - 1);
    else if (i == b.ni) tcol = load_target(a.faces, b.face_off[3], j - 1);
    const int gstage = (*a.iter) * 4 + a.stage + 1;
#pragma unroll
    for (int n = 0; n < P; ++n) {
        // hbcore.py:197-221: stencil, then m ascending (D[n][n] = +0 included
        // as its exact 0*q product), then the forcing term
        double o = stencil(cur[n], wv[n], ev[n], sv_[n], nv[n], b.nu_h2, b.adv_2h);
#pragma unroll
        for (int m = 0; m < P; ++m) o = radd(o, rmul(a.D[n * P + m], cur[m]));
        o = radd(o, rmul(a.ap[n * NPDE + p], sv));
        const double v = rsub(bq[n], rmul(a.coef, o));
        double *dst = a.out + cell + n * ps4;
        if (sector_store) {
            double2 *sec = reinterpret_cast<double2 *>((uintptr_t)dst & ~(uintptr_t)31);
            const int pos = (int)(((uintptr_t)dst >> 3) & 3);
            sec[0] = make_double2(pos == 0 ? v : 0.0, pos == 1 ? v : 0.0);
            sec[1] = make_double2(pos == 2 ? v : 0.0, pos == 3 ? v : 0.0);
        } else {
            *dst = v;
        }
        forward(trow, a.out, a.sendbuf, n, p, v);
        forward(tcol, a.out, a.sendbuf, n, p, v);
        if (nonfinite(v)) {
            const long long lin = (((long long)(n * NPDE + p) * b.nj + (j - 1)) * b.ni) + (i - 1);
            atomicMin(a.status + sg.block, divergence_key(gstage, lin));
        }
    }
}

template <int P>
static int launch_band(const hbgpu_stage_args &a, cudaStream_t s) {
    // dir-2 segments cover 64 rows per block, others 128 cells
    const dim3 grid((unsigned)((a.band_max_len + 63) / 64), (unsigned)a.nband_segs, NPDE);
    band_kernel<P><<<grid, 128, 0, s>>>(a);
    hbgpu_count_launch(1);
    return hbgpu_check_launch("hbgpu_band");
}

// ---- the paired stage kernel ------------------------------------------------------
//
// CTA structure as stage_tma_kernel (hb_stage.cu) -- 8 consumer warps, a
// TMA load warp, a TMA store warp -- plus an edge warp (v1 at the strip's
// edge columns); tiles of 256/PT columns x PT pdes x tile_rows rows;
// lane = column.  Per row step r the consumers
//   1. compute v1(r), the pair's first stage, from the stencil ring (rows
//      r-1, r, r+1 of `in`, all read from shared memory);
//   2. publish v1(r) in a 3-row shared ring and meet on a named barrier;
//   3. compute v2(r-1), the second stage, from v1 rows r-2..r of their own
//      column (registers) and v1(r-1) of the neighbouring columns (the
//      shared ring, or -- at the strip's two edge columns -- the band slot's
//      granules that ride on the stencil row's TMA transaction).
// v1 above / below the tile (rows j0-1, j1+1) is read from the band slot.
// Pass A (stages 0, 1) stores v2 with plain stores and forwards south/north
// face rows; pass B (stages 2, 3) stages v2 in the q0 slot it replaces for
// the TMA store warp and forwards nothing (a full halo pass follows).
// Requires every block's ni to be a multiple of the strip width (all lanes
// live); the engine falls back to single stages otherwise.

template <int P, bool PB, int R, int Q, int PT>
struct PairSmem {
    using G = Geo<PT>;
    static constexpr int BOXD = P * PT * G::BW;
    static constexpr int REGION = (BOXD * 8 + 127) / 128 * 128 / 8;
    static constexpr int EDGE = (P * PT * 8 * 8 + 127) / 128 * 128 / 8;   // {8 cols, PT, P} granule box
    static constexpr int EDGE_W = G::NSPLIT * REGION;                     // band v1, column i0-1
    static constexpr int EDGE_E = EDGE_W + EDGE;                          // band v1, column i0+TCOLS
    static constexpr int SXY = EDGE_E + EDGE;
    static constexpr int SLOT = SXY + G::TCOLS;
    static constexpr int QSLOT = P * PT * G::TCOLS;
    static constexpr int NQ = PB ? Q : 0;
    static constexpr int NV = 3;                                          // v1 rows in flight
    // a v1 row holds, per (plane, pde), the strip's columns plus the two edge
    // columns i0-1 (index 0) and i0+TCOLS (index TCOLS+1), which the edge
    // warp writes: every consumer lane then reads its west / east v1
    // neighbour at the same compile-time offsets
    static constexpr int VPITCH = G::TCOLS + 2;
    static constexpr int VROW = P * PT * VPITCH;
    static constexpr size_t V1_OFF = ((size_t)R * SLOT + (size_t)NQ * QSLOT) * 8;
    static constexpr size_t BAR_OFF = V1_OFF + ((size_t)NV * VROW * 8 + 15) / 16 * 16;
    static constexpr size_t BYTES = BAR_OFF + (size_t)(2 * R + 3 * NQ) * 8;
    static_assert((SLOT * 8) % 128 == 0 && (QSLOT * 8) % 128 == 0, "TMA slots need 128-B alignment");
};

// Three warpgroups: the 8 consumer warps (two groups) and a helper group of
// the TMA load warp, the TMA store warp, the edge warp and one idle warp.
// The helpers need few registers: after the launch (168 per thread) the
// helper group gives registers back (setmaxnreg.dec) and the consumer groups
// take them (setmaxnreg.inc), so the consumers can hold two register row
// windows (the input rows r-1..r+1 and v1 rows r-2..r) without spilling.
constexpr int PAIR_THREADS = (CW + 4) * 32;
static_assert(CW == 8, "two consumer warpgroups + one helper warpgroup");
// per tile geometry: the PT = 4 edge warp carries 3 (side, pde, plane)
// items per lane and needs more registers.  Budget: 256 * (consumer - 168)
// <= 128 * (168 - helper) + (65536 - 384 * 168).
#ifndef HBGPU_PAIR_HELPER_REGS   // measurement builds may move the split
#define HBGPU_PAIR_HELPER_REGS 72
#endif
#ifndef HBGPU_PAIR_CONSUMER_REGS
#define HBGPU_PAIR_CONSUMER_REGS 208
#endif
template <int PT> struct PairRegs {
    static constexpr int HELPER = PT == 1 ? HBGPU_PAIR_HELPER_REGS : 80;
    static constexpr int CONSUMER = PT == 1 ? HBGPU_PAIR_CONSUMER_REGS : 208;
    static_assert(256 * (CONSUMER - 168) <= 128 * (168 - HELPER) + (65536 - PAIR_THREADS * 168), "regs");
};

template <int PT>
__device__ __forceinline__ void helper_regs() {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(PairRegs<PT>::HELPER));
}
template <int PT>
__device__ __forceinline__ void consumer_regs() {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(PairRegs<PT>::CONSUMER));
}

// the consumers and the edge warp meet once per row step (v1(r) of every
// column, the edge columns included, is in the v1 ring) and at each tile end
__device__ __forceinline__ void consumer_sync() {
    asm volatile("bar.sync 1, %0;" ::"n"((HBGPU_TILE_WARPS + 1) * 32) : "memory");
}

// o = residual, v = base - coef * o: the reference's per-point rounding
// sequence (hbcore.py:197-221, 240) with two exact rewrites that the paired
// schedule's eligibility guarantees (devlayout.fused_eligible: nu_h2 >= 1)
// and the hazard keys police (record_nonfinite):
//
// 1. t = 4c - w as one DFMA.  4c is exact (a power-of-two scaling) unless it
//    overflows, i.e. unless |c| >= 2^1022, so round(4c - w) == the
//    reference's round(round(4c) - w).  Every value this library writes is
//    checked: one of magnitude >= 2^1022 records a hazard key, and the run
//    is repeated on the strict single-stage kernels (solver.run_case), so a
//    result that depended on an overflowing 4c is never returned.
//
// 2. The signed-zero terms -- D[n][n]*q[n] (D[n][n] = +0) and the forcing of
//    the unforced planes (amplitude +0) -- are dropped.  Adding +-0 to o
//    changes o only when o == -0, and o is never -0 here: with nu_h2 >= 1,
//    t*nu_h2 is -0 only if t is (no underflow to zero), t is -0 only if
//    4c == -0 and w, e, s, n are all +0, and then (e - w)*adv_2h is +0, so
//    t*nu_h2 + u is not -0; a round-to-nearest sum is -0 only when both
//    addends are, so no later partial sum is -0 either.
template <int P>
__device__ __forceinline__ void stage_point(const double (&c)[P], const double (&w)[P], const double (&e)[P],
                                            const double (&s)[P], const double (&nn)[P], const double (&dk)[P / 2 + 1],
                                            const double (&ap)[P], double sv, double nu_h2, double adv_2h,
                                            double coef, const double (&base)[P], double (&o)[P], double (&v)[P]) {
#pragma unroll
    for (int n = 0; n < P; ++n) o[n] = __fma_rn(4.0, c[n], -w[n]);
#pragma unroll
    for (int n = 0; n < P; ++n) o[n] = rsub(o[n], e[n]);
#pragma unroll
    for (int n = 0; n < P; ++n) o[n] = rsub(o[n], s[n]);
#pragma unroll
    for (int n = 0; n < P; ++n) o[n] = rsub(o[n], nn[n]);
#pragma unroll
    for (int n = 0; n < P; ++n) o[n] = rmul(o[n], nu_h2);
#pragma unroll
    for (int n = 0; n < P; ++n) o[n] = radd(o[n], rmul(rsub(e[n], w[n]), adv_2h));
#pragma unroll
    for (int m = 0; m < P; ++m) {
#pragma unroll
        for (int k = 1; k <= P / 2; ++k) {
            const double prod = rmul(dk[k], c[m]);
            o[(m + k) % P] = radd(o[(m + k) % P], prod);
            o[(m + P - k) % P] = rsub(o[(m + P - k) % P], prod);
        }
    }
#pragma unroll
    for (int n = 0; n < P; ++n) {
        if (forced_plane(n)) o[n] = radd(o[n], rmul(ap[n], sv));
        v[n] = rsub(base[n], rmul(coef, o[n]));
    }
}

template <int P>
__device__ __forceinline__ void record_nonfinite(const double (&v)[P], const hbgpu_stage_args &a, int bidx,
                                                 const hbgpu_block &b, int p, int j, int i, int gstage) {
    // on the integer pipe (the fp64 pipe is this kernel's binding resource):
    // the largest masked exponent field of the P values is >= 0x7fd iff one
    // of them is non-finite (0x7ff: a divergence key) or has magnitude
    // >= 2^1022 (a hazard key: stage_point's DFMA 4c - w would not be the
    // reference's rounding for it in the next stage)
    unsigned ex = 0;
#pragma unroll
    for (int n = 0; n < P; ++n) ex = max(ex, (unsigned)__double2hiint(v[n]) & 0x7ff00000u);
    if (ex >= HAZARD_EXP) {
        for (int n = 0; n < P; ++n) {
            const unsigned e = (unsigned)__double2hiint(v[n]) & 0x7ff00000u;
            if (e < HAZARD_EXP) continue;
            const long long lin = (((long long)(n * NPDE + p) * b.nj + (j - 1)) * b.ni) + (i - 1);
            atomicMin(a.status + bidx, e == 0x7ff00000u ? divergence_key(gstage, lin) : hazard_key(gstage, lin));
        }
    }
}

template <int P, bool PB, int R, int Q, int PT>
__global__ void __launch_bounds__(PAIR_THREADS, 1) pair_tma_kernel(const __grid_constant__ hbgpu_stage_args a) {
    using S = PairSmem<P, PB, R, Q, PT>;
    using G = Geo<PT>;
    static_assert(R >= 4 && (!PB || Q >= 3), "ring too short");
    extern __shared__ __align__(1024) unsigned char smem[];
    double *ring = reinterpret_cast<double *>(smem);
    double *qring = ring + R * S::SLOT;
    double *v1ring = reinterpret_cast<double *>(smem + S::V1_OFF);
    uint64_t *full_in = reinterpret_cast<uint64_t *>(smem + S::BAR_OFF);
    uint64_t *empty_in = full_in + R;
    uint64_t *full_q = empty_in + R;
    uint64_t *empty_q = full_q + S::NQ;   // q0 slot stored out and free (store warp)
    uint64_t *staged = empty_q + S::NQ;   // v2 row written over it (consumers)
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int k = 0; k < R; ++k) {
            mbar_init(full_in + k, 1);
            mbar_init(empty_in + k, CW + 1);   // consumers + the edge warp
        }
        for (int k = 0; k < S::NQ; ++k) {
            mbar_init(full_q + k, 1);
            mbar_init(empty_q + k, 1);
            mbar_init(staged + k, CW * 32);
        }
        fence_mbar_init();
    }
    __syncthreads();
    const int ntile = tile_end(a);
    const CUtensorMap *maps = reinterpret_cast<const CUtensorMap *>(a.tmaps);
    const bool inter = a.interleaved != 0;
    if (warp >= CW) {
        helper_regs<PT>();
        if (warp == CW + 3) return;   // the helper group's fourth warp
    }

    if (warp == CW) {
        // ------------------------------ producer ------------------------------
        if (lane != 0) return;
        constexpr uint32_t BYTES = S::BOXD * 8 * G::NSPLIT, QBYTES = S::QSLOT * 8, SBYTES = G::TCOLS * 8,
                           EBYTES = P * PT * 8 * 8;
        RingPos pin{0, 0}, pq{0, 0};
        int issued_in = 0, issued_q = 0;
        for (int k = a.tile_lo + blockIdx.x; k < ntile; k += gridDim.x) {
            const int t = tile_at(a, k);
            const Tile tl = decode_tile<PT>(a, t);
            const CUtensorMap *min = maps + a.in_slot * a.nblocks + tl.bidx;
            const CUtensorMap *mq = maps + 3 * a.nblocks + tl.bidx;
            const CUtensorMap *ms = maps + 4 * a.nblocks + tl.bidx;
            const CUtensorMap *me = maps + 9 * a.nblocks + tl.bidx;   // band slot, one granule
            prefetch_tmap(min);
            const int x = tl.i0 + LEAD - 2;
            const int west_face = tl.i0 == 1, east_face = tl.i0 + G::TCOLS > a.blocks[tl.bidx].ni;
            // entry of row `row`: the stencil row, sxy of row-1 (with_sxy) and
            // the band values at the strip's two edge columns (with_edge)
            auto put_in = [&](int row, bool with_sxy, bool with_edge) {
                if (issued_in >= R) mbar_wait_idle(empty_in + pin.slot, pin.phase ^ 1u);
                else ++issued_in;
                double *dst = ring + pin.slot * S::SLOT;
                mbar_expect_tx(full_in + pin.slot, BYTES + (with_sxy ? SBYTES : 0) +
                                                       (with_edge ? (west_face + east_face) * EBYTES : 0));
#pragma unroll
                for (int k = 0; k < G::NSPLIT; ++k)
                    load_rows<PT>(dst + k * S::REGION, min, x + k * (G::TCOLS / G::NSPLIT), tl.pde0, row, inter,
                                  full_in + pin.slot);
                if (with_sxy) tma_load_2d(dst + S::SXY, ms, tl.i0 - 1, row - 2, full_in + pin.slot);
                // a strip edge on a block face reads the band slot's halo (TMA);
                // an edge inside the block is computed by the edge warp
                if (with_edge && west_face)
                    load_rows<PT>(dst + S::EDGE_W, me, tl.i0 + LEAD - 8, tl.pde0, row, inter, full_in + pin.slot);
                if (with_edge && east_face)
                    load_rows<PT>(dst + S::EDGE_E, me, tl.i0 + LEAD + G::TCOLS, tl.pde0, row, inter,
                                  full_in + pin.slot);
                pin = advance<R>(pin);
            };
            put_in(tl.j0 - 1, false, false);
            put_in(tl.j0, false, true);
            for (int j = tl.j0; j <= tl.j1; ++j) {
                put_in(j + 1, true, j + 1 <= tl.j1);
                if (PB) {
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
    if (warp == CW + 1) {
        // ----------------------- store warp (pass B only) -----------------------
        if (!PB || lane != 0) return;
        RingPos ps{0, 0};
        for (int k = a.tile_lo + blockIdx.x; k < ntile; k += gridDim.x) {
            const int t = tile_at(a, k);
            const Tile tl = decode_tile<PT>(a, t);
            const CUtensorMap *mo = maps + (5 + a.out_slot) * a.nblocks + tl.bidx;
            prefetch_tmap(mo);
            for (int j = tl.j0; j <= tl.j1; ++j) {
                mbar_wait_idle(staged + ps.slot, ps.phase);
                store_rows(mo, qring + ps.slot * S::QSLOT, tl.i0 + LEAD, tl.pde0, j, inter);
                bulk_commit();
                bulk_wait_read_all();
                mbar_arrive(empty_q + ps.slot);
                ps = advance<Q>(ps);
            }
        }
        bulk_wait_all();
        return;
    }

    if (warp == CW + 2) {
        // ------------------------------ edge warp ------------------------------
        // v1 of the strip's two edge columns (i0-1, i0+TCOLS), written into
        // the v1 ring's edge columns before the row step's barrier:
        //  * inside the block, lane k = (side, pde, plane n) accumulates plane
        //    n's residual in the reference order (hbcore.py:197-221: stencil,
        //    m ascending, forcing) from the stencil slots;
        //  * on a block face, v1 is the band slot's halo value, which the
        //    producer's TMA brought into the row's slot as an edge granule.
        // The south value of each item is kept from the previous row step, so
        // row r's slot is released as soon as row r's v1 is written: the
        // consumers and this warp free a slot one row earlier than a
        // three-row stencil read would, and the ring looks one row further.
        constexpr int NE = 2 * PT * P;
        constexpr int KE = (NE + 31) / 32;   // (side, pde, plane) items per lane
        // per item: its plane's D row and forcing amplitude (fixed), and the
        // forcing / q0 values of the next row, loaded one row ahead
        double drow[KE][P];
        int side_k[KE], pp_k[KE], n_k[KE], off_k[KE], vcol_k[KE], gran_k[KE];
#pragma unroll
        for (int c = 0; c < KE; ++c) {
            const int k = lane + 32 * c;
            side_k[c] = k < NE ? k / (PT * P) : 2;
            pp_k[c] = (k / P) % PT;
            n_k[c] = k % P;
            const int side = side_k[c], pp = pp_k[c], n = n_k[c];
            // smem column of the edge cell inside the stencil box
            const int region = side == 0 ? 0 : G::NSPLIT - 1;
            const int idx = side == 0 ? 1 : G::TCOLS - region * (G::TCOLS / G::NSPLIT) + 2;
            off_k[c] = region * S::REGION + pp * G::BW + idx + n * PT * G::BW;
            vcol_k[c] = (n * PT + pp) * S::VPITCH + (side == 0 ? 0 : G::TCOLS + 1);
            gran_k[c] = side == 0 ? S::EDGE_W + (n * PT + pp) * 8 + 7 : S::EDGE_E + (n * PT + pp) * 8;
#pragma unroll
            for (int m = 0; m < P; ++m) drow[c][m] = k < NE ? a.D[n * P + m] : 0.0;
        }
        RingPos cin{0, 0};
        int vr = 0;   // v1 ring row of v1(r), in step with the consumers
        for (int k = a.tile_lo + blockIdx.x; k < ntile; k += gridDim.x) {
            const int t = tile_at(a, k);
            const Tile tl = decode_tile<PT>(a, t);
            const hbgpu_block b = a.blocks[tl.bidx];
            const bool west_in = tl.i0 > 1, east_in = tl.i0 + G::TCOLS <= b.ni;
            const int64_t erow = (int64_t)t * a.tile_rows;   // this tile's rows in edge_q0
            bool act[KE], live[KE];
            int ie_k[KE];
            double ap_k[KE], sv_n[KE], bs_n[KE], south[KE];
#pragma unroll
            for (int c = 0; c < KE; ++c) {
                live[c] = side_k[c] < 2;
                act[c] = side_k[c] == 0 ? west_in : side_k[c] == 1 ? east_in : false;
                ie_k[c] = side_k[c] == 0 ? tl.i0 - 1 : tl.i0 + G::TCOLS;
                ap_k[c] = act[c] ? a.ap[n_k[c] * NPDE + tl.pde0 + pp_k[c]] : 0.0;
            }
            auto fetch = [&](int rr) {
#pragma unroll
                for (int c = 0; c < KE; ++c) {
                    if (!act[c]) continue;
                    sv_n[c] = __ldg(a.sxy + b.sxy_off + (int64_t)(rr - 1) * b.sxy_pitch + (ie_k[c] - 1));
                    // q0 at the edge cell: pass B overwrites q0 in place, and the
                    // edge column belongs to the neighbouring strip, whose CTA
                    // may already have replaced it -- read pass A's copy
                    if (PB) bs_n[c] = __ldg(a.edge_q0 + (erow + rr - tl.j0) * NE + lane + 32 * c);
                }
            };
            fetch(tl.j0);
            {
                // row j0-1: only its centre values are used (v1(j0)'s south)
                mbar_wait_idle(full_in + cin.slot, cin.phase);
                const double *ru = ring + cin.slot * S::SLOT;
#pragma unroll
                for (int c = 0; c < KE; ++c)
                    if (act[c]) south[c] = ru[off_k[c]];
                __syncwarp();
                if (lane == 0) mbar_arrive(empty_in + cin.slot);
                cin = advance<R>(cin);
            }
            for (int r = tl.j0; r <= tl.j1; ++r) {
                double sv_c[KE], bs_c[KE];
#pragma unroll
                for (int c = 0; c < KE; ++c) {
                    sv_c[c] = sv_n[c];
                    bs_c[c] = bs_n[c];
                }
                if (r < tl.j1) fetch(r + 1);
                const RingPos nx = advance<R>(cin);
                // row r as the previous step's row r+1, except at the tile's
                // first row: the ring's fills complete in any order, so row
                // j0+1 having landed says nothing about row j0
                if (r == tl.j0) mbar_wait_idle(full_in + cin.slot, cin.phase);
                mbar_wait_idle(full_in + nx.slot, nx.phase);
                const double *rc = ring + cin.slot * S::SLOT;
                const double *rn = ring + nx.slot * S::SLOT;
                double *vrow = v1ring + vr * S::VROW;
#pragma unroll
                for (int c = 0; c < KE; ++c) {
                    if (!live[c]) continue;
                    double v;
                    if (act[c]) {
                        const double *cc = rc + off_k[c];
                        const double cen = cc[0];
                        double o = stencil(cen, cc[-1], cc[1], south[c], rn[off_k[c]], b.nu_h2, b.adv_2h);
                        const double *cm = rc + off_k[c] - n_k[c] * PT * G::BW;   // plane 0 of the column
#pragma unroll
                        for (int m = 0; m < P; ++m) o = radd(o, rmul(drow[c][m], cm[m * PT * G::BW]));
                        o = radd(o, rmul(ap_k[c], sv_c[c]));
                        const double base = PB ? bs_c[c] : cen;
                        if (!PB) a.edge_q0[(erow + r - tl.j0) * NE + lane + 32 * c] = base;   // q0 (pass A: in)
                        v = rsub(base, rmul(a.coef, o));
                        south[c] = cen;
                    } else {
                        v = rc[gran_k[c]];   // block face: the band slot's halo value
                    }
                    vrow[vcol_k[c]] = v;
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(empty_in + cin.slot);   // row r: read for the last time
                consumer_sync();   // the consumers' barrier of row step r
                cin = nx;
                vr = vr == S::NV - 1 ? 0 : vr + 1;
            }
            // row j1+1 was read as the last row's north only
            __syncwarp();
            if (lane == 0) mbar_arrive(empty_in + cin.slot);
            consumer_sync();   // the consumers' tile-end barrier
            cin = advance<R>(cin);
        }
        return;
    }

    // -------------------------------- consumers ---------------------------------
    // (every helper warp has returned above: this region runs at CONSUMER_REGS)
    consumer_regs<PT>();
    const int pp = warp % PT;
    const int cw = warp / PT;
    const int col0 = 32 * cw + lane;
    const int in_off = (cw / G::CWPR) * S::REGION + pp * G::BW + 32 * (cw % G::CWPR) + lane + 2;
    const int q_off = pp * G::TCOLS + col0;
    // this lane's column in a v1 ring row; its west / east v1 neighbours for
    // the second stage sit at -1 / +1 (the edge warp's columns at the strip's
    // edges)
    const int v_off = pp * S::VPITCH + 1 + col0;
    const int gstage = (*a.iter) * 4 + a.stage + 1;   // first stage of the pair; +1 for the second
    const double coef1 = a.coef, coef2 = a.coef2;
    double dk[P / 2 + 1];
#pragma unroll
    for (int k = 1; k <= P / 2; ++k) dk[k] = a.D[k * P];
    RingPos cin{0, 0}, cq{0, 0};
    int ap_pde = -1;
    double ap[P];
    int vr = 0;   // v1 ring row of v1(r)
    for (int k = a.tile_lo + blockIdx.x; k < ntile; k += gridDim.x) {
            const int t = tile_at(a, k);
        const Tile tl = decode_tile<PT>(a, t);
        const int p = tl.pde0 + pp;
        if (p != ap_pde) {
#pragma unroll
            for (int n = 0; n < P; ++n) ap[n] = a.ap[n * NPDE + p];
            ap_pde = p;
        }
        const hbgpu_block b = a.blocks[tl.bidx];
        const double nu_h2 = b.nu_h2, adv_2h = b.adv_2h;
        // stage_point's dropped signed zeros need nu_h2 >= 1 (the engine only
        // pairs such blocks; a C-ABI caller that does not gets a hazard key,
        // i.e. "repeat on the strict kernels")
        if (warp == 0 && lane == 0 && !(nu_h2 >= 1.0)) atomicMin(a.status + tl.bidx, hazard_key(gstage, 0));
        const int i = tl.i0 + col0;
        const int64_t ps4 = b.ps * NPDE;
        const int64_t colbase = b.base + (int64_t)p * b.ps + LEAD + i;   // (n=0, p, j=0, i)
        // v1 of row j0-1 (band slot: the neighbouring row tile's perimeter
        // row, or the block's halo row)
        double va[P], vb[P], vc[P];
#pragma unroll
        for (int n = 0; n < P; ++n) vb[n] = __ldg(a.band + colbase + n * ps4 + (int64_t)(tl.j0 - 1) * b.rs);
        double nrm = 0.0;
        double sv_prev = 0.0;
        // input window: this lane's column of `in` at rows r-1, r, r+1 stays
        // in registers, so a row step loads only the new row's centre and
        // the current row's west / east neighbours from the ring
        double xa[P], xb[P], xc[P];
        {
            // row j0-1 entry: only its centre row is used (as v1(j0)'s south)
            const RingPos cu = cin;
            cin = advance<R>(cin);
            mbar_wait(full_in + cu.slot, cu.phase);
            mbar_wait(full_in + cin.slot, cin.phase);
            const double *ru = ring + cu.slot * S::SLOT + in_off;
            const double *rc = ring + cin.slot * S::SLOT + in_off;
#pragma unroll
            for (int n = 0; n < P; ++n) {
                xa[n] = ru[n * PT * G::BW];
                xb[n] = rc[n * PT * G::BW];
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(empty_in + cu.slot);   // row j0-1: read for the last time
        }
        // one row step: v1(r) and, one row behind, v2(r-1).  Input window on
        // entry: ia = in(r-1), ib = in(r); ic <- in(r+1)
        auto row_step = [&](const int r, double(&pa)[P], double(&pb)[P], double(&pc)[P], double(&ia)[P],
                            double(&ib)[P], double(&ic)[P]) {
            // rows r-1 and r were waited for as earlier steps' rows r and r+1
            // (the tile's first step: before the first step)
            const RingPos nx = advance<R>(cin);
            mbar_wait(full_in + nx.slot, nx.phase);
            const double *rc = ring + cin.slot * S::SLOT + in_off;
            const double *rn = ring + nx.slot * S::SLOT + in_off;
            const double sv = ring[nx.slot * S::SLOT + S::SXY + col0];
            const double *qv = nullptr;
            if (PB) {
                mbar_wait(full_q + cq.slot, cq.phase);
                qv = qring + cq.slot * S::QSLOT + q_off;
            }
            double o[P], v[P];
            {
                double w[P], e[P], base[P];
#pragma unroll
                for (int n = 0; n < P; ++n) {
                    ic[n] = rn[n * PT * G::BW];
                    w[n] = rc[n * PT * G::BW - 1];
                    e[n] = rc[n * PT * G::BW + 1];
                    base[n] = PB ? qv[n * PT * G::TCOLS] : ib[n];
                }
                stage_point<P>(ib, w, e, ia, ic, dk, ap, sv, nu_h2, adv_2h, coef1, base, o, pc);
            }
            if (!PB) {
#pragma unroll
                for (int n = 0; n < P; ++n) nrm = __fma_rn(o[n], o[n], nrm);
            }
            record_nonfinite<P>(pc, a, tl.bidx, b, p, r, i, gstage);
            double *vrow = v1ring + vr * S::VROW + v_off;
#pragma unroll
            for (int n = 0; n < P; ++n) vrow[n * PT * S::VPITCH] = pc[n];
            consumer_sync();
            if (r > tl.j0) {
                // second stage at row r-1
                const int vp = vr == 0 ? S::NV - 1 : vr - 1;   // v1 ring row of v1(r-1)
                const double *vv = v1ring + vp * S::VROW + v_off;
                double w2[P], e2[P], base2[P];
#pragma unroll
                for (int n = 0; n < P; ++n) {
                    w2[n] = vv[n * PT * S::VPITCH - 1];
                    e2[n] = vv[n * PT * S::VPITCH + 1];
                }
                if (PB) {
                    // q0 of row r-1: the previous q slot
                    const RingPos cqp = cq.slot == 0 ? RingPos{Q - 1, cq.phase ^ 1u} : RingPos{cq.slot - 1, cq.phase};
                    const double *qp = qring + cqp.slot * S::QSLOT + q_off;
#pragma unroll
                    for (int n = 0; n < P; ++n) base2[n] = qp[n * PT * G::TCOLS];
                    stage_point<P>(pb, w2, e2, pa, pc, dk, ap, sv_prev, nu_h2, adv_2h, coef2, base2, o, v);
                    double *stage_row = qring + cqp.slot * S::QSLOT + q_off;
#pragma unroll
                    for (int n = 0; n < P; ++n) stage_row[n * PT * G::TCOLS] = v[n];
                    fence_proxy_async_smem();
                    mbar_arrive(staged + cqp.slot);
                } else {
#pragma unroll
                    for (int n = 0; n < P; ++n) base2[n] = ia[n];   // q0 = in, row r-1
                    stage_point<P>(pb, w2, e2, pa, pc, dk, ap, sv_prev, nu_h2, adv_2h, coef2, base2, o, v);
                    const int64_t row = (int64_t)(r - 1) * b.rs;
#pragma unroll
                    for (int n = 0; n < P; ++n) a.out[colbase + n * ps4 + row] = v[n];
                }
                record_nonfinite<P>(v, a, tl.bidx, b, p, r - 1, i, gstage + 1);
            }
            sv_prev = sv;
            __syncwarp();
            if (lane == 0) mbar_arrive(empty_in + cin.slot);   // row r no longer read
            cin = nx;
            if (PB) cq = advance<Q>(cq);
            vr = vr == S::NV - 1 ? 0 : vr + 1;
        };
        // v1 window (pa, pb) = (v1(r-2), v1(r-1)) on entry of step r; pc <- v1(r)
        int r = tl.j0;
        for (; r + 2 <= tl.j1; r += 3) {
            row_step(r, va, vb, vc, xa, xb, xc);
            row_step(r + 1, vb, vc, va, xb, xc, xa);
            row_step(r + 2, vc, va, vb, xc, xa, xb);
        }
        // last second-stage row: v2(j1) from the window (A, B) = (v1(j1-1),
        // v1(j1)) and v1(j1+1) from the band slot; X = in(j1) (pass A: q0
        // row j1)
        auto last_step = [&](double(&A)[P], double(&B)[P], double(&X)[P]) {
            double vd[P];
#pragma unroll
            for (int n = 0; n < P; ++n) vd[n] = __ldg(a.band + colbase + n * ps4 + (int64_t)(tl.j1 + 1) * b.rs);
            const int vp = vr == 0 ? S::NV - 1 : vr - 1;   // v1 ring row of v1(j1)
            const double *vv = v1ring + vp * S::VROW + v_off;
            double w2[P], e2[P], base2[P], o[P], v[P];
#pragma unroll
            for (int n = 0; n < P; ++n) {
                w2[n] = vv[n * PT * S::VPITCH - 1];
                e2[n] = vv[n * PT * S::VPITCH + 1];
            }
            if (PB) {
                const RingPos cqp = cq.slot == 0 ? RingPos{Q - 1, cq.phase ^ 1u} : RingPos{cq.slot - 1, cq.phase};
                const double *qp = qring + cqp.slot * S::QSLOT + q_off;
#pragma unroll
                for (int n = 0; n < P; ++n) base2[n] = qp[n * PT * G::TCOLS];
                stage_point<P>(B, w2, e2, A, vd, dk, ap, sv_prev, nu_h2, adv_2h, coef2, base2, o, v);
                double *stage_row = qring + cqp.slot * S::QSLOT + q_off;
#pragma unroll
                for (int n = 0; n < P; ++n) stage_row[n * PT * G::TCOLS] = v[n];
                fence_proxy_async_smem();
                mbar_arrive(staged + cqp.slot);
            } else {
#pragma unroll
                for (int n = 0; n < P; ++n) base2[n] = X[n];
                stage_point<P>(B, w2, e2, A, vd, dk, ap, sv_prev, nu_h2, adv_2h, coef2, base2, o, v);
                const int64_t row = (int64_t)tl.j1 * b.rs;
#pragma unroll
                for (int n = 0; n < P; ++n) a.out[colbase + n * ps4 + row] = v[n];
            }
            record_nonfinite<P>(v, a, tl.bidx, b, p, tl.j1, i, gstage + 1);
        };
        if (r > tl.j1) {
            last_step(va, vb, xa);
        } else if (r == tl.j1) {
            row_step(r, va, vb, vc, xa, xb, xc);
            last_step(vb, vc, xb);
        } else {
            row_step(r, va, vb, vc, xa, xb, xc);
            row_step(r + 1, vb, vc, va, xb, xc, xa);
            last_step(vc, va, xc);
        }
        if (!PB) {
            // pass A forwards the block's south / north face rows (a full halo
            // pass follows pass B).  Out of the row loop: the lane reads back
            // the v2 values it stored itself (same thread, program order) for
            // the at most two face rows of the tile, instead of testing for a
            // face row in every row step.
            auto forward_row = [&](int j) {
                const FaceHit trow = row_target(a.faces, b, i, j, true);
                if (trow.ps == 0) return;
                double v[P];
#pragma unroll
                for (int n = 0; n < P; ++n) v[n] = a.out[colbase + n * ps4 + (int64_t)j * b.rs];
#pragma unroll
                for (int n = 0; n < P; ++n) forward(trow, a.out, a.sendbuf, n, p, v[n]);
            };
            if (tl.j0 == 1) forward_row(1);
            if (tl.j1 == b.nj && b.nj > 1) forward_row(b.nj);
        }
        // every consumer is past its reads of the v1 ring before the next
        // tile's first row overwrites it
        consumer_sync();
        __syncwarp();
        if (lane == 0) mbar_arrive(empty_in + cin.slot);   // row j1+1 (row j1 left with its row step)
        cin = advance<R>(cin);
        if (!PB && a.norm_part != nullptr) {
            const double s = warp_sum(nrm);
            if (lane == 0) a.norm_part[(int64_t)t * CW + warp] = s;
        }
    }
}

// ---- launch ---------------------------------------------------------------------

struct PairLaunch {
    void (*fn)(hbgpu_stage_args) = nullptr;
    size_t smem = 0;
    int grid = 0;
    bool ready = false;
};

template <int P, bool PB, int R, int Q, int PT>
static int prepare_pair(PairLaunch &L) {
    if (L.ready) return HBGPU_OK;
    L.fn = pair_tma_kernel<P, PB, R, Q, PT>;
    L.smem = PairSmem<P, PB, R, Q, PT>::BYTES;
    if (cudaFuncSetAttribute(L.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.smem) != cudaSuccess)
        return hbgpu_check_launch("pair kernel smem attribute");
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, L.fn, PAIR_THREADS, L.smem) != cudaSuccess ||
        per_sm < 1)
        return hbgpu_check_launch("pair kernel occupancy");
    L.grid = sms * per_sm;
    L.ready = true;
    return HBGPU_OK;
}

// ring depths: pass A has no q0 ring, so its stencil ring can go one deeper
// (two rows of look-ahead); pass B fits R = 4 with a 4-deep q0 ring
#ifndef HBGPU_PAIR_RA
#define HBGPU_PAIR_RA 5
#endif
#ifndef HBGPU_PAIR_R
#define HBGPU_PAIR_R 4
#endif
#ifndef HBGPU_PAIR_Q
#define HBGPU_PAIR_Q 4
#endif

template <int P, int PT>
static int pair_cfg(const hbgpu_stage_args &a, cudaStream_t s, bool prepare_only) {
    // the smem attribute and the occupancy grid are per device
    static PairLaunch la_d[HB_MAX_DEVICES], lb_d[HB_MAX_DEVICES];
    const int dev = current_device();
    if (dev < 0) return HBGPU_ERR_CUDA;
    PairLaunch &la = la_d[dev], &lb = lb_d[dev];
    int rc = prepare_pair<P, false, HBGPU_PAIR_RA, HBGPU_PAIR_Q, PT>(la);
    if (!rc) rc = prepare_pair<P, true, HBGPU_PAIR_R, HBGPU_PAIR_Q, PT>(lb);
    if (rc || prepare_only) return rc;
    if (a.tmaps == nullptr || a.band == nullptr || a.edge_q0 == nullptr) {
        hbgpu_set_error("hbgpu_stage (pair): args->tmaps, args->band and args->edge_q0 are required");
        return HBGPU_ERR_ARG;
    }
    PairLaunch &L = a.pair == 2 ? lb : la;
    const int grid = persistent_grid(L.grid, tile_end(a) - a.tile_lo);
    L.fn<<<grid, PAIR_THREADS, L.smem, s>>>(a);
    hbgpu_count_launch(1);
    return hbgpu_check_launch("hbgpu_stage (pair)");
}

template <int P>
static int pair_p(const hbgpu_stage_args &a, cudaStream_t s, bool prepare_only) {
    return a.tile_pdes == 1 ? pair_cfg<P, 1>(a, s, prepare_only) : pair_cfg<P, 4>(a, s, prepare_only);
}

int pair_dispatch(const hbgpu_stage_args &a, cudaStream_t s, bool prepare_only) {
    switch (a.planes) {
        case 1: return pair_p<1>(a, s, prepare_only);
        case 3: return pair_p<3>(a, s, prepare_only);
        case 5: return pair_p<5>(a, s, prepare_only);
        case 7: return pair_p<7>(a, s, prepare_only);
        case 9: return pair_p<9>(a, s, prepare_only);
        default: break;
    }
    // the stencil ring, the v1 ring and the q0 ring of pass B fit the 227 KB
    // of shared memory up to P = 9
    hbgpu_set_error("paired stages need P <= %d, got %d", HBGPU_MAX_PAIR_P, a.planes);
    return HBGPU_ERR_UNSUPPORTED;
}

}  // namespace hbgpu

extern "C" int hbgpu_band(const hbgpu_stage_args *a, void *stream) {
    using namespace hbgpu;
    if (a == nullptr || a->nband_segs < 0 || a->nband_segs > 65535 || a->band_max_len < 0) {
        hbgpu_set_error("hbgpu_band: bad arguments");
        return HBGPU_ERR_ARG;
    }
    if (a->nband_segs == 0 || a->band_max_len == 0) return HBGPU_OK;
    cudaStream_t s = (cudaStream_t)stream;
    switch (a->planes) {
        case 1: return launch_band<1>(*a, s);
        case 3: return launch_band<3>(*a, s);
        case 5: return launch_band<5>(*a, s);
        case 7: return launch_band<7>(*a, s);
        case 9: return launch_band<9>(*a, s);
        case 11: return launch_band<11>(*a, s);
        case 13: return launch_band<13>(*a, s);
        case 15: return launch_band<15>(*a, s);
        case 17: return launch_band<17>(*a, s);
        default: break;
    }
    hbgpu_set_error("hbgpu_band: P=%d is above the templated range (%d)", a->planes, HBGPU_MAX_TEMPLATED_P);
    return HBGPU_ERR_UNSUPPORTED;
}
