// hb_aux.cu -- the small kernels around the stage kernel:
//   * standalone halo moves (priming exchange, unpack, exchange_halos);
//   * residual-norm folding;
//   * force integration and the rank-ordered fold;
//   * the kernel-level drop-ins for _residual_kernel / _update_kernel on the
//     reference's dense (planes, npde, nj+2, ni+2) layout.

#include "hb_common.cuh"

namespace hbgpu {

// ---- halo moves (exchange.py:195-202, 248-261) ------------------------------

// One thread per (direction, element, slice of the 4P values).  Consecutive
// threads take consecutive elements, so a row face (element stride 1) moves
// as coalesced 256-byte warp accesses; a column face is one cell per row,
// and its slot-halo destination is written as the cell's whole 32-byte
// sector (HBGPU_HALO_SECTOR_DST: the rest of the sector is row lead or
// padding) so L2 never fills a partial sector.  Each thread keeps up to 8
// loads in flight.
constexpr int HALO_THREADS = 128;
constexpr int HALO_VCHUNK = 8;

__global__ void __launch_bounds__(HALO_THREADS) halo_kernel(double *slot, double *sendbuf, const double *recvbuf,
                                                            const hbgpu_halo_dir *dirs, int nv) {
    const hbgpu_halo_dir d = dirs[blockIdx.y];
    const int64_t e = (int64_t)blockIdx.x * HALO_THREADS + threadIdx.x;
    if (e >= d.length) return;
    const int v0 = blockIdx.z * HALO_VCHUNK;
    const int nvk = min(HALO_VCHUNK, nv - v0);
    const double *src = (d.src_kind == 0 ? slot : (d.src_kind == 1 ? sendbuf : recvbuf)) + d.src_off + e * d.src_es;
    double *dst = (d.dst_kind == 0 ? slot : sendbuf) + d.dst_off + e * d.dst_es;
    double val[HALO_VCHUNK];
#pragma unroll
    for (int k = 0; k < HALO_VCHUNK; ++k)
        if (k < nvk) val[k] = src[(int64_t)(v0 + k) * d.src_vs];
    const bool sector = (d.flags & HBGPU_HALO_SECTOR_DST) != 0 && d.dst_kind == 0;
#pragma unroll
    for (int k = 0; k < HALO_VCHUNK; ++k) {
        if (k >= nvk) break;
        double *t = dst + (int64_t)(v0 + k) * d.dst_vs;
        if (sector) {
            double2 *sec = reinterpret_cast<double2 *>((uintptr_t)t & ~(uintptr_t)31);
            const int pos = (int)(((uintptr_t)t >> 3) & 3);
            sec[0] = make_double2(pos == 0 ? val[k] : 0.0, pos == 1 ? val[k] : 0.0);
            sec[1] = make_double2(pos == 2 ? val[k] : 0.0, pos == 3 ? val[k] : 0.0);
        } else {
            *t = val[k];
        }
    }
}

// ---- hazard scan ----------------------------------------------------------------

// Any finite value of magnitude >= 2^1022 in a block's region of `slot` sets
// the block's hazard key at gstage 0 (before the first stage): the paired
// kernel's DFMA 4c - w matches the reference only below that (hb_pair.cu
// stage_point).  Regions are 256-B aligned and a multiple of 8 elements.
__global__ void hazard_scan_kernel(const double *slot, const hbgpu_block *blocks, int planes,
                                   unsigned long long *status) {
    const hbgpu_block b = blocks[blockIdx.y];
    const int64_t n2 = (int64_t)planes * NPDE * (b.nj + 2) * b.pitch / 2;
    const double2 *p = reinterpret_cast<const double2 *>(slot + b.base);
    unsigned ex = 0;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n2; k += (int64_t)gridDim.x * blockDim.x) {
        const double2 v = p[k];
        const unsigned e0 = (unsigned)__double2hiint(v.x) & 0x7ff00000u, e1 = (unsigned)__double2hiint(v.y) & 0x7ff00000u;
        if (e0 >= HAZARD_EXP && e0 != 0x7ff00000u) ex = 1;
        if (e1 >= HAZARD_EXP && e1 != 0x7ff00000u) ex = 1;
    }
    if (__any_sync(0xffffffffu, ex != 0) && (threadIdx.x & 31) == 0) atomicMin(status + blockIdx.y, hazard_key(0, 0));
}

// ---- residual norm ----------------------------------------------------------

// per block: one CTA folds its (tile, consumer warp) partials -- thread t
// takes partials t, t + NF, t + 2 NF, ... in order, then a fixed-shape tree
// over the threads.  Deterministic for a given tile layout (the norm is not a
// reference quantity; the oracle's fsum agrees to rtol 1e-12).  sumsq holds
// max_iters rows: an iteration counter at or past it writes nothing.
constexpr int NF_THREADS = 256;

__global__ void __launch_bounds__(NF_THREADS) norm_fold_kernel(const hbgpu_block *blocks, int nblocks,
                                                               const double *part, double *sumsq,
                                                               const int32_t *iter, int max_iters) {
    __shared__ double red[NF_THREADS];
    const int b = blockIdx.x;
    const int it = *iter;
    if (b >= nblocks || it >= max_iters || it < 0) return;
    const hbgpu_block &blk = blocks[b];
    // one partial per (tile, consumer warp), tiles of a block contiguous
    constexpr int W = HBGPU_TILE_WARPS;
    const int64_t n = (int64_t)blk.ntiles * W;
    const double *p = part + (int64_t)blk.tile_begin * W;
    double s = 0.0;
    for (int64_t c = threadIdx.x; c < n; c += NF_THREADS) s = radd(s, p[c]);
    red[threadIdx.x] = s;
    __syncthreads();
    for (int w = NF_THREADS / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) red[threadIdx.x] = radd(red[threadIdx.x], red[threadIdx.x + w]);
        __syncthreads();
    }
    if (threadIdx.x == 0) sumsq[(int64_t)it * nblocks + b] = red[0];
}

// one thread per iteration: the rank-global per-block sums of R^2 (columns in
// ascending global block id) folded left to right, then the correctly
// rounded square root -- bitwise the host's math.sqrt(sum(...)) fold
__global__ void norm_totals_kernel(const double *sumsq, int iters, int nblocks, double *norms) {
    const int it = blockIdx.x * blockDim.x + threadIdx.x;
    if (it >= iters) return;
    double s = 0.0;
    for (int b = 0; b < nblocks; ++b) s = radd(s, sumsq[(int64_t)it * nblocks + b]);
    norms[it] = __dsqrt_rn(s);
}

// ---- forces (hbcore.py:359-382) --------------------------------------------

// One warp per (coefficient k, plane n, body) output: a strict left-to-right
// fold of h*q over the body's face segments in reference order.  The warp
// loads the face in chunks of FCH cells (lanes on consecutive cells, the next
// chunk's loads in flight during the fold), forms the products h*q in
// parallel (each rounded once, as in the reference), and lane 0 adds them in
// order from shared memory -- the fold itself is the only serial part.  Then
// one thread advances the device iteration counter (this is the iteration's
// last kernel).  hist holds max_iters rows; an iteration counter at or past
// it writes no history (the engine refuses to issue such iterations anyway).
constexpr int FORCE_WARPS = 32;
constexpr int FCH = 128;
constexpr int FU = FCH / 32;

__global__ void __launch_bounds__(FORCE_WARPS * 32) forces_kernel(const double *slot, const hbgpu_force_seg *segs,
                                                                  int nsegs, int planes, int nbody, double *hist,
                                                                  int32_t *iter, int max_iters) {
    __shared__ double prod[FORCE_WARPS][FCH];
    const int it = *iter;
    const int total = (it >= 0 && it < max_iters) ? 3 * planes * nbody : 0;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
    double *buf = prod[warp];
    for (int t = warp; t < total; t += nwarps) {
        const int body = t % nbody;
        const int n = (t / nbody) % planes;
        const int k = t / (nbody * planes);
        double acc = 0.0;
        for (int s = 0; s < nsegs; ++s) {
            const hbgpu_force_seg g = segs[s];
            if (g.body != body) continue;
            const double *f = slot + g.start + (int64_t)(n * NPDE + k) * g.ps;
            double v[FU];
#pragma unroll
            for (int u = 0; u < FU; ++u) {
                const int c = lane + 32 * u;
                v[u] = c < g.length ? f[(int64_t)c * g.stride] : 0.0;
            }
            for (int c0 = 0; c0 < g.length; c0 += FCH) {
#pragma unroll
                for (int u = 0; u < FU; ++u) buf[lane + 32 * u] = rmul(g.h, v[u]);
                __syncwarp();
#pragma unroll
                for (int u = 0; u < FU; ++u) {
                    const int c = c0 + FCH + lane + 32 * u;
                    v[u] = c < g.length ? f[(int64_t)c * g.stride] : 0.0;
                }
                if (lane == 0) {
                    const int m = min(FCH, g.length - c0);
                    int e = 0;
                    for (; e + 8 <= m; e += 8) {
#pragma unroll
                        for (int u = 0; u < 8; ++u) acc = radd(acc, buf[e + u]);
                    }
                    for (; e < m; ++e) acc = radd(acc, buf[e]);
                }
                __syncwarp();
            }
        }
        if (lane == 0) hist[(int64_t)it * total + t] = acc;
    }
    __syncthreads();
    if (threadIdx.x == 0) *iter = it + 1;
}

// runtime.py:290-294: acc = buf[0]; acc += buf[1]; ...
__global__ void ordered_fold_kernel(const double *stacked, int nranks, int64_t count, double *out) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= count) return;
    double acc = stacked[k];
    for (int r = 1; r < nranks; ++r) acc = radd(acc, stacked[(int64_t)r * count + k]);
    out[k] = acc;
}

// ---- dense-layout drop-ins -------------------------------------------------

struct Dense {
    int64_t planes, npde, nj2, ni2;
    __device__ int64_t q(int64_t n, int64_t p, int64_t j, int64_t i) const {
        return ((n * npde + p) * nj2 + j) * ni2 + i;
    }
    __device__ int64_t r(int64_t n, int64_t p, int64_t j, int64_t i) const {
        return ((n * npde + p) * (nj2 - 2) + j) * (ni2 - 2) + i;
    }
};

__global__ void residual_dense_kernel(const double *q, const double *dmat, const double *src,
                                      double nu_h2, double adv_2h, double *out, Dense d,
                                      int64_t n_lo, int64_t n_hi, int64_t j_lo, int64_t j_hi) {
    const int64_t ni = d.ni2 - 2;
    const int64_t rows = j_hi - j_lo;
    const int64_t total = (n_hi - n_lo) * d.npde * rows * ni;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = t % ni + 1;
        int64_t rest = t / ni;
        const int64_t j = rest % rows + j_lo;
        rest /= rows;
        const int64_t p = rest % d.npde;
        const int64_t n = rest / d.npde + n_lo;
        const double *c = q + d.q(n, p, j, i);
        double o = stencil(c[0], c[-1], c[1], c[-d.ni2], c[d.ni2], nu_h2, adv_2h);
        for (int64_t m = 0; m < d.planes; ++m)
            o = radd(o, rmul(dmat[n * d.planes + m], q[d.q(m, p, j, i)]));
        o = radd(o, src[d.r(n, p, j - 1, i - 1)]);
        out[d.r(n, p, j - 1, i - 1)] = o;
    }
}

// snapshot (all columns of the rows, halo columns included) and update
// (interior); each element depends only on itself, so one pass suffices.
__global__ void update_dense_kernel(double *q, double *q0, const double *resid, double coef,
                                    int snapshot, Dense d, int64_t n_lo, int64_t n_hi,
                                    int64_t j_lo, int64_t j_hi, unsigned long long *first_bad) {
    const int64_t ni = d.ni2 - 2, nj = d.nj2 - 2;
    const int64_t rows = j_hi - j_lo;
    const int64_t total = (n_hi - n_lo) * d.npde * rows * d.ni2;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = t % d.ni2;
        int64_t rest = t / d.ni2;
        const int64_t j = rest % rows + j_lo;
        rest /= rows;
        const int64_t p = rest % d.npde;
        const int64_t n = rest / d.npde + n_lo;
        const int64_t k = d.q(n, p, j, i);
        if (snapshot) q0[k] = q[k];
        if (i == 0 || i == d.ni2 - 1) continue;
        const double v = rsub(q0[k], rmul(coef, resid[d.r(n, p, j - 1, i - 1)]));
        q[k] = v;
        if (nonfinite(v))
            atomicMin(first_bad, (unsigned long long)((((n * d.npde + p) * nj) + (j - 1)) * ni + (i - 1)));
    }
}

__global__ void first_nonfinite_kernel(const double *q, Dense d, unsigned long long *first_bad) {
    const int64_t ni = d.ni2 - 2, nj = d.nj2 - 2;
    const int64_t total = d.planes * d.npde * nj * ni;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = t % ni;
        int64_t rest = t / ni;
        const int64_t j = rest % nj;
        const int64_t np = rest / nj;
        if (nonfinite(q[(np * d.nj2 + j + 1) * d.ni2 + i + 1])) atomicMin(first_bad, (unsigned long long)t);
    }
}

static int grid_for(int64_t total) {
    int64_t g = (total + 255) / 256;
    if (g > 148 * 64) g = 148 * 64;
    return (int)(g < 1 ? 1 : g);
}

}  // namespace hbgpu

using namespace hbgpu;

extern "C" int hbgpu_halo(double *slot, double *sendbuf, const double *recvbuf,
                          const hbgpu_halo_dir *dirs, int32_t ndirs, int32_t max_len,
                          int32_t planes, void *stream) {
    if (ndirs <= 0 || max_len <= 0) return HBGPU_OK;
    const int nv = planes * NPDE;
    dim3 grid((unsigned)((max_len + HALO_THREADS - 1) / HALO_THREADS), (unsigned)ndirs,
              (unsigned)((nv + HALO_VCHUNK - 1) / HALO_VCHUNK));
    halo_kernel<<<grid, HALO_THREADS, 0, (cudaStream_t)stream>>>(slot, sendbuf, recvbuf, dirs, nv);
    hbgpu_count_launch(1);
    return hbgpu_check_launch("hbgpu_halo");
}

extern "C" int hbgpu_hazard_scan(const double *slot, const hbgpu_block *blocks, int32_t nblocks, int32_t planes,
                                 unsigned long long *status, void *stream) {
    if (nblocks <= 0) return HBGPU_OK;
    if (nblocks > 65535) {
        hbgpu_set_error("hbgpu_hazard_scan: %d blocks exceed one grid row per block", nblocks);
        return HBGPU_ERR_ARG;
    }
    hazard_scan_kernel<<<dim3(64, (unsigned)nblocks), 256, 0, (cudaStream_t)stream>>>(slot, blocks, planes, status);
    hbgpu_count_launch(1);
    return hbgpu_check_launch("hbgpu_hazard_scan");
}

extern "C" int hbgpu_norm_totals(const double *sumsq, int32_t iters, int32_t nblocks, double *norms,
                                 void *stream) {
    if (iters <= 0) return HBGPU_OK;
    norm_totals_kernel<<<(iters + 127) / 128, 128, 0, (cudaStream_t)stream>>>(sumsq, iters, nblocks, norms);
    hbgpu_count_launch(1);
    return hbgpu_check_launch("hbgpu_norm_totals");
}

extern "C" int hbgpu_norm_fold(const hbgpu_block *blocks, int32_t nblocks, const double *norm_part,
                               double *sumsq, const int32_t *iter, int32_t max_iters, void *stream) {
    if (nblocks <= 0) return HBGPU_OK;
    if (nblocks > 65535) {
        hbgpu_set_error("hbgpu_norm_fold: %d blocks exceed one CTA per block", nblocks);
        return HBGPU_ERR_ARG;
    }
    norm_fold_kernel<<<(unsigned)nblocks, NF_THREADS, 0, (cudaStream_t)stream>>>(blocks, nblocks, norm_part, sumsq,
                                                                                iter, max_iters);
    hbgpu_count_launch(1);
    return hbgpu_check_launch("hbgpu_norm_fold");
}

extern "C" int hbgpu_forces(const double *slot, const hbgpu_force_seg *segs, int32_t nsegs,
                            int32_t planes, int32_t nbody, double *hist, int32_t *iter, int32_t max_iters,
                            void *stream) {
    int warps = 3 * planes * nbody;
    warps = warps < 1 ? 1 : (warps > FORCE_WARPS ? FORCE_WARPS : warps);
    forces_kernel<<<1, warps * 32, 0, (cudaStream_t)stream>>>(slot, segs, nsegs, planes, nbody, hist, iter,
                                                           max_iters);
    hbgpu_count_launch(1);
    return hbgpu_check_launch("hbgpu_forces");
}

extern "C" int hbgpu_ordered_fold(const double *stacked, int32_t nranks, int64_t count, double *out,
                                  void *stream) {
    if (count <= 0) return HBGPU_OK;
    ordered_fold_kernel<<<(unsigned)((count + 127) / 128), 128, 0, (cudaStream_t)stream>>>(stacked, nranks,
                                                                                        count, out);
    hbgpu_count_launch(1);
    return hbgpu_check_launch("hbgpu_ordered_fold");
}

extern "C" int hbgpu_residual(const double *q, const double *dmat, const double *src, double nu_h2,
                              double adv_2h, double *out, int64_t planes, int64_t npde, int64_t nj2,
                              int64_t ni2, int64_t n_lo, int64_t n_hi, int64_t j_lo, int64_t j_hi,
                              void *stream) {
    if (n_hi <= n_lo || j_hi <= j_lo || ni2 < 3) return HBGPU_OK;
    Dense d{planes, npde, nj2, ni2};
    const int64_t total = (n_hi - n_lo) * npde * (j_hi - j_lo) * (ni2 - 2);
    residual_dense_kernel<<<grid_for(total), 256, 0, (cudaStream_t)stream>>>(q, dmat, src, nu_h2, adv_2h,
                                                                           out, d, n_lo, n_hi, j_lo, j_hi);
    hbgpu_count_launch(1);
    return hbgpu_check_launch("hbgpu_residual");
}

extern "C" int hbgpu_update(double *q, double *q0, const double *resid, double coef, int snapshot,
                            int64_t planes, int64_t npde, int64_t nj2, int64_t ni2, int64_t n_lo,
                            int64_t n_hi, int64_t j_lo, int64_t j_hi, unsigned long long *first_bad,
                            void *stream) {
    if (n_hi <= n_lo || j_hi <= j_lo) return HBGPU_OK;
    Dense d{planes, npde, nj2, ni2};
    const int64_t total = (n_hi - n_lo) * npde * (j_hi - j_lo) * ni2;
    update_dense_kernel<<<grid_for(total), 256, 0, (cudaStream_t)stream>>>(q, q0, resid, coef, snapshot, d,
                                                                         n_lo, n_hi, j_lo, j_hi, first_bad);
    hbgpu_count_launch(1);
    return hbgpu_check_launch("hbgpu_update");
}

extern "C" int hbgpu_first_nonfinite(const double *q, int64_t planes, int64_t npde, int64_t nj2,
                                     int64_t ni2, unsigned long long *first_bad, void *stream) {
    Dense d{planes, npde, nj2, ni2};
    const int64_t total = planes * npde * (nj2 - 2) * (ni2 - 2);
    first_nonfinite_kernel<<<grid_for(total), 256, 0, (cudaStream_t)stream>>>(q, d, first_bad);
    hbgpu_count_launch(1);
    return hbgpu_check_launch("hbgpu_first_nonfinite");
}
