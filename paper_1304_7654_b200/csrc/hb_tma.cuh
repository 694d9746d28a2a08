// hb_tma.cuh -- device helpers shared by the stage kernels (hb_stage.cu,
// hb_pair.cu): mbarrier / tensor-TMA PTX wrappers, the strip geometry, tile
// decoding, halo-target forwarding and ring positions.
#pragma once

#include "hb_common.cuh"

#include <cuda.h>

namespace hbgpu {

// ---- PTX: mbarrier + tensor TMA --------------------------------------------------

__device__ __forceinline__ uint32_t saddr(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(saddr(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(saddr(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(b)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t parity) {
    uint32_t done;
    do {
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(done)
            : "r"(saddr(b)), "r"(parity)
            : "memory");
    } while (!done);
}
// The same wait for the helper warps (TMA load / store, edge): the thread
// asks to be suspended until the phase completes (up to the hint, in ns)
// instead of re-polling, so a producer running rows ahead does not take
// issue slots from the consumer warps sharing its scheduler.
__device__ __forceinline__ void mbar_wait_idle(uint64_t *b, uint32_t parity) {
    uint32_t done;
    do {
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3; selp.u32 %0, 1, 0, p; }"
            : "=r"(done)
            : "r"(saddr(b)), "r"(parity), "n"(1000000)
            : "memory");
    } while (!done);
}
__device__ __forceinline__ void tma_load_4d(void *dst, const void *map, int c0, int c1, int c2, int c3,
                                            uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(saddr(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(saddr(bar))
        : "memory");
}
__device__ __forceinline__ void tma_load_2d(void *dst, const void *map, int c0, int c1, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(saddr(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(saddr(bar))
        : "memory");
}
__device__ __forceinline__ void tma_store_4d(const void *map, int c0, int c1, int c2, int c3, const void *src) {
    asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4}], [%5];" ::"l"(map),
                 "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(saddr(src))
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// wait until every committed bulk store has finished READING shared memory
__device__ __forceinline__ void bulk_wait_read_all() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
// make this thread's generic-proxy shared-memory writes visible to TMA
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void prefetch_tmap(const void *map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(map) : "memory");
}

// ---- geometry ---------------------------------------------------------------------

constexpr int CW = HBGPU_TILE_WARPS;            // consumer warps per tile
constexpr int THREADS = (CW + 2) * 32;          // + one TMA load warp + one TMA store warp
// Tile geometry for PT pdes per tile (4 or 1).
template <int PT>
struct Geo {
    static constexpr int TCOLS = 256 / PT;                     // strip columns
    static constexpr int NSPLIT = (TCOLS + 4 > 256) ? 2 : 1;   // stencil boxes per row
    static constexpr int BW = TCOLS / NSPLIT + 4;              // stencil box width
    static constexpr int CWPR = TCOLS / 32 / NSPLIT;           // column warps per box
    static_assert(PT == 1 || PT == 4, "tile_pdes is 1 or 4");
    static_assert(BW <= 256, "TMA box limit");
};

// Interior columns 1..store_cols(ni) of a row go out by TMA store; the rest
// (at most 7, ni not a multiple of 8) by plain stores.  The store tensor map
// ends on a 64-B boundary: a bulk store may write whole granules, and the
// granule holding cell ni also holds the east halo cell ni+1, which the
// neighbouring block's tile forwards into concurrently.
__host__ __device__ __forceinline__ int store_cols(int ni) { return ni / 8 * 8; }

// ---- tiles and halo targets -------------------------------------------------

struct Tile {
    int bidx;   // local block index
    int i0;     // first interior column of the strip (1-based)
    int pde0;   // first pde of the tile
    int j0, j1; // first / last interior row
};

template <int PT>
__device__ __forceinline__ Tile decode_tile(const hbgpu_stage_args &a, int t) {
    Tile T;
    T.bidx = a.tile_block[t];
    const hbgpu_block &b = a.blocks[T.bidx];
    const int local = t - b.tile_begin;
    T.i0 = (local % b.tiles_i) * Geo<PT>::TCOLS + 1;
    const int rest = local / b.tiles_i;
    constexpr int GROUPS = NPDE / PT;
    T.pde0 = (rest % GROUPS) * PT;
    T.j0 = (rest / GROUPS) * a.tile_rows + 1;
    T.j1 = min(T.j0 + a.tile_rows - 1, b.nj);
    return T;
}

// the launch's tile range (hbgpu_stage_args.tile_order / tile_lo / tile_hi):
// persistent CTAs walk k = tile_lo + blockIdx.x, += gridDim.x, below
// tile_end(a), processing tile tile_at(a, k)
__host__ __device__ __forceinline__ int tile_end(const hbgpu_stage_args &a) {
    return a.tile_hi > 0 ? a.tile_hi : a.total_tiles;
}
__device__ __forceinline__ int tile_at(const hbgpu_stage_args &a, int k) {
    return a.tile_order != nullptr ? a.tile_order[k] : k;
}

struct FaceHit {
    int64_t off;
    int64_t ps;
};

__device__ __forceinline__ FaceHit load_target(const hbgpu_face_target *pool, int64_t base, int k) {
    FaceHit t{0, 0};
    if (base >= 0) {
        hbgpu_face_target v = pool[base + k];
        t.off = v.off;
        t.ps = v.ps;
    }
    return t;
}

// halo targets of cell (i, j): the south/north face target and the west/east one
__device__ __forceinline__ void cell_targets(const hbgpu_face_target *pool, const hbgpu_block &b, int i,
                                             int j, bool live, FaceHit &trow, FaceHit &tcol) {
    trow = FaceHit{0, 0};
    tcol = FaceHit{0, 0};
    if (!live) return;
    if (j == 1) trow = load_target(pool, b.face_off[0], i - 1);
    else if (j == b.nj) trow = load_target(pool, b.face_off[1], i - 1);
    if (i == 1) tcol = load_target(pool, b.face_off[2], j - 1);
    else if (i == b.ni) tcol = load_target(pool, b.face_off[3], j - 1);
}

// the south/north face target of cell (i, j)
__device__ __forceinline__ FaceHit row_target(const hbgpu_face_target *pool, const hbgpu_block &b, int i, int j,
                                              bool live) {
    if (!live) return FaceHit{0, 0};
    if (j == 1) return load_target(pool, b.face_off[0], i - 1);
    if (j == b.nj) return load_target(pool, b.face_off[1], i - 1);
    return FaceHit{0, 0};
}

__device__ __forceinline__ void forward(const FaceHit &t, double *out, double *sendbuf, int n, int p,
                                        double v) {
    constexpr int64_t SECTOR = (int64_t)1 << HBGPU_SECTOR_TARGET_BIT;
    if (t.ps > 0) {
        double *dst = out + (t.off & ~SECTOR) + (int64_t)(n * NPDE + p) * t.ps;
        if (t.off & SECTOR) {
            // the whole 32-byte sector: the value in place, zeros in the lead /
            // padding around it (no partial-sector fill in L2)
            double2 *sec = reinterpret_cast<double2 *>((uintptr_t)dst & ~(uintptr_t)31);
            const int pos = (int)(((uintptr_t)dst >> 3) & 3);
            sec[0] = make_double2(pos == 0 ? v : 0.0, pos == 1 ? v : 0.0);
            sec[1] = make_double2(pos == 2 ? v : 0.0, pos == 3 ? v : 0.0);
        } else {
            *dst = v;
        }
    } else if (t.ps < 0) {
        sendbuf[t.off + n * NPDE + p] = v;
    }
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = radd(v, __shfl_down_sync(0xffffffffu, v, o));
    return v;
}

// ---- ring positions -----------------------------------------------------------------

struct RingPos {
    int slot;
    uint32_t phase;   // mbarrier phase parity of the slot's current fill
};

template <int N>
__device__ __forceinline__ RingPos advance(RingPos r) {
    if (++r.slot == N) {
        r.slot = 0;
        r.phase ^= 1u;
    }
    return r;
}

// TMA coordinates of (column x, first pde, row) for either slot layout
template <int PT>
__device__ __forceinline__ void load_rows(void *dst, const void *map, int x, int pde0, int row, bool inter,
                                          uint64_t *bar) {
    if (inter) tma_load_4d(dst, map, x, pde0, 0, row, bar);
    else tma_load_4d(dst, map, x, row, pde0, 0, bar);
}
__device__ __forceinline__ void store_rows(const void *map, const void *src, int x, int pde0, int row, bool inter) {
    if (inter) tma_store_4d(map, x, pde0, 0, row, src);
    else tma_store_4d(map, x, row, pde0, 0, src);
}

// Persistent grid of a stage / pair launch: min(resident CTAs, tiles),
// further capped by HBGPU_GRID_LIMIT when set (a test knob: with a few CTAs
// each one walks many tiles, which exercises the rings' tile-to-tile hand-
// over and lets strips drift apart as they do at full size).
int persistent_grid(int resident, int tiles);

// launch configurations (smem attribute, occupancy grid) are cached per
// device ordinal; current_device() is the cache index, -1 on error
constexpr int HB_MAX_DEVICES = 64;
int current_device();

// hb_pair.cu: launch (or, prepare_only, just configure) the paired-stage
// kernel for args.pair = 1 (stages 0, 1) or 2 (stages 2, 3)
int pair_dispatch(const hbgpu_stage_args &a, cudaStream_t s, bool prepare_only);

}  // namespace hbgpu
