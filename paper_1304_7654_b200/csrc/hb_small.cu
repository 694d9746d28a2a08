// hb_small.cu -- whole iterations of a small single-GPU rank in one launch.
//
// For a small rank (BASELINE C0/C1: up to a few MB per slot, L2-resident)
// the per-stage TMA kernels spend most of their time in launch, pipeline
// fill and drain.  Here one cooperative launch runs `iters` complete
// iterations: the 4 RK stages, separated by grid-wide barriers.  Each stage
// is one flat task list over every block of the rank -- a warp task is
// (block, row, pde, 32-column chunk), a thread computes one (cell, pde) for
// all P planes -- strided over all warps of the grid, with
//   * halo forwarding at write time through the face-target pool (local
//     cut halo cells of the output slot; the rank has no remote cuts),
//   * divergence keys per block (hbcore.py:279-284),
//   * stage 0: per warp task a fixed shuffle tree, per (warp, block) the
//     warp's tasks in order, per (CTA, block) the warps in order; at stage 1
//     one warp per block folds the CTA partials (lane-strided, fixed shuffle
//     tree) -- deterministic for a given grid,
//   * forces of each iteration into the history after the last stage: one
//     warp per (coefficient, plane, body), the products h*q formed by the
//     whole warp and folded left to right by lane 0 (the next iteration's
//     first stage only reads slot A, so the other warps go on),
// and the iteration counter set once at the end.  Operands come through L1
// and L2; every rounding is the reference's (strict rmul/radd, the signed
// zero terms included), so the fields equal the other schedules' bitwise.

#include "hb_tma.cuh"

#include <cooperative_groups.h>
#include <string.h>

#include <algorithm>
#include <vector>

namespace cg = cooperative_groups;

namespace hbgpu {

constexpr int SMALL_THREADS = 256;
constexpr int SMALL_WARPS = SMALL_THREADS / 32;
constexpr int SMALL_MAX_BLOCKS = 256;   // task offsets live in shared memory
constexpr int SMALL_FCH = 128;          // force chunk per warp
constexpr int SMALL_MAX_CTAS = 4096;    // grid cap (the per-(CTA, block) partials)
// slot rotation (hb_runtime.cu kIn / kOut): A -> B -> C -> B -> A
__device__ __forceinline__ int in_slot_of(int st) { return st == 0 ? 0 : (st == 2 ? 2 : 1); }
__device__ __forceinline__ int out_slot_of(int st) { return st == 3 ? 0 : (st == 1 ? 2 : 1); }

struct SmallArgs {
    double *slot[3];
    const hbgpu_block *blocks;
    const double *sxy;
    const hbgpu_face_target *faces;
    unsigned long long *status;
    int32_t *iter;
    double *sumsq;           // [max_iters * nblocks]
    double *task_part;       // [gridDim.x * nblocks] stage-0 partials per (CTA, block)
    const hbgpu_force_seg *segs;
    double *force_hist;      // [max_iters * 3 * planes * nbody]
    int32_t nblocks, planes, nbody, nsegs;
    int32_t it0, iters, max_iters, pad;
    double coef[4];
    double D[HBGPU_MAX_TEMPLATED_P * HBGPU_MAX_TEMPLATED_P];
    double ap[HBGPU_MAX_TEMPLATED_P * HBGPU_NPDE];
};

// One (cell, pde) with all P planes: the P centres serve the coupling sum
// of every plane, each plane's neighbours are loaded once; all 6P + 1 loads
// are independent (issued together).  Returns the sum of R^2 over the planes.
template <int P>
__device__ __forceinline__ double small_cell(const SmallArgs &a, const hbgpu_block &b, const double *in,
                                             const double *q0, double *out, int st, int p, int j, int i, int gstage,
                                             int bidx) {
    const int64_t ps4 = b.ps * NPDE;
    const int64_t cell = b.base + (int64_t)p * b.ps + (int64_t)j * b.rs + LEAD + i;
    const double *c = in + cell;
    double cur[P], wv[P], ev[P], sv_[P], nv[P], bq[P];
#pragma unroll
    for (int m = 0; m < P; ++m) {
        const double *cm = c + m * ps4;
        cur[m] = __ldg(cm);
        wv[m] = __ldg(cm - 1);
        ev[m] = __ldg(cm + 1);
        sv_[m] = __ldg(cm - b.rs);
        nv[m] = __ldg(cm + b.rs);
        bq[m] = st == 0 ? cur[m] : q0[cell + m * ps4];
    }
    const double sv = __ldg(a.sxy + b.sxy_off + (int64_t)(j - 1) * b.sxy_pitch + (i - 1));
    FaceHit trow, tcol;
    cell_targets(a.faces, b, i, j, true, trow, tcol);
    const double coef = a.coef[st];
    double acc = 0.0;
#pragma unroll
    for (int n = 0; n < P; ++n) {
        // hbcore.py:197-221: stencil, m ascending (D[n][n] = +0 as its exact
        // 0*q product), forcing; hbcore.py:240: q0 - coef*R
        double o = stencil(cur[n], wv[n], ev[n], sv_[n], nv[n], b.nu_h2, b.adv_2h);
#pragma unroll
        for (int m = 0; m < P; ++m) o = radd(o, rmul(a.D[n * P + m], cur[m]));
        o = radd(o, rmul(a.ap[n * NPDE + p], sv));
        const double v = rsub(bq[n], rmul(coef, o));
        out[cell + n * ps4] = v;
        forward(trow, out, nullptr, n, p, v);
        forward(tcol, out, nullptr, n, p, v);
        acc = __fma_rn(o, o, acc);
        if (nonfinite(v)) {
            const long long lin = (((long long)(n * NPDE + p) * b.nj + (j - 1)) * b.ni) + (i - 1);
            atomicMin(a.status + bidx, divergence_key(gstage, lin));
        }
    }
    return acc;
}

template <int P>
struct SmallBounds {
    // P <= 7 fits 128 registers (two CTAs per SM); P = 9 keeps its loads in
    // flight with up to 255 (one CTA)
    static constexpr int MIN_BLOCKS = P <= 7 ? 2 : 1;
};

template <int P>
__global__ void __launch_bounds__(SMALL_THREADS, SmallBounds<P>::MIN_BLOCKS)
    small_kernel(const __grid_constant__ SmallArgs a) {
    cg::grid_group grid = cg::this_grid();
    __shared__ int task_off[SMALL_MAX_BLOCKS + 1];
    __shared__ int chunks_of[SMALL_MAX_BLOCKS];
    __shared__ double fbuf[SMALL_WARPS][SMALL_FCH];
    __shared__ double red[SMALL_WARPS][SMALL_MAX_BLOCKS];
    const int lane = threadIdx.x & 31;
    const int nwarps = gridDim.x * SMALL_WARPS;
    const int gwarp = blockIdx.x * SMALL_WARPS + (threadIdx.x >> 5);
    if (threadIdx.x == 0) {
        // warp tasks of block b: (row, pde, 32-column chunk), chunk fastest
        int off = 0;
        for (int b = 0; b < a.nblocks; ++b) {
            const int chunks = (a.blocks[b].ni + 31) >> 5;
            chunks_of[b] = chunks;
            task_off[b] = off;
            off += chunks * NPDE * a.blocks[b].nj;
        }
        task_off[a.nblocks] = off;
    }
    __syncthreads();
    const int tasks = task_off[a.nblocks];
    const int total_f = 3 * P * a.nbody;
    for (int it = 0; it < a.iters; ++it) {
        const int iter = a.it0 + it;
        for (int st = 0; st < 4; ++st) {
            const double *in = a.slot[in_slot_of(st)];
            const double *q0 = a.slot[0];
            double *out = a.slot[out_slot_of(st)];
            const int gstage = iter * 4 + st + 1;
            if (st == 1 && gwarp < a.nblocks && iter < a.max_iters) {
                // this iteration's stage-0 partials of block gwarp: CTAs
                // lane-strided in order (8 loads in flight), then a fixed
                // shuffle tree
                double s = 0.0;
                const int nc = gridDim.x;
                for (int c0 = lane; c0 < nc; c0 += 32 * 8) {
                    double v[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const int c = c0 + 32 * u;
                        v[u] = c < nc ? a.task_part[(int64_t)c * a.nblocks + gwarp] : 0.0;
                    }
#pragma unroll
                    for (int u = 0; u < 8; ++u)
                        if (c0 + 32 * u < nc) s = radd(s, v[u]);
                }
                for (int o = 16; o > 0; o >>= 1) s = radd(s, __shfl_down_sync(0xffffffffu, s, o));
                if (lane == 0) a.sumsq[(int64_t)iter * a.nblocks + gwarp] = s;
            }
            const int wib = threadIdx.x >> 5;
            if (st == 0) {
                for (int k = threadIdx.x; k < SMALL_WARPS * a.nblocks; k += SMALL_THREADS)
                    red[k / a.nblocks][k % a.nblocks] = 0.0;
                __syncthreads();
            }
            int bidx = 0, cur_b = -1;
            double acc_b = 0.0;
            for (int t = gwarp; t < tasks; t += nwarps) {
                while (t >= task_off[bidx + 1]) ++bidx;   // tasks ascend per warp
                const hbgpu_block &b = a.blocks[bidx];
                const int chunks = chunks_of[bidx];
                const int r = t - task_off[bidx];
                const int chunk = r % chunks;
                const int pj = r / chunks;
                const int p = pj % NPDE, j = pj / NPDE + 1;
                const int i = (chunk << 5) + lane + 1;
                double acc = 0.0;
                if (i <= b.ni) acc = small_cell<P>(a, b, in, q0, out, st, p, j, i, gstage, bidx);
                if (st == 0) {
                    for (int o = 16; o > 0; o >>= 1) acc = radd(acc, __shfl_down_sync(0xffffffffu, acc, o));
                    if (bidx != cur_b) {
                        if (cur_b >= 0 && lane == 0) red[wib][cur_b] = acc_b;
                        acc_b = 0.0;
                        cur_b = bidx;
                    }
                    acc_b = radd(acc_b, acc);
                }
            }
            if (st == 0) {
                if (cur_b >= 0 && lane == 0) red[wib][cur_b] = acc_b;
                __syncthreads();
                for (int bb = threadIdx.x; bb < a.nblocks; bb += SMALL_THREADS) {
                    double s = 0.0;
                    for (int w2 = 0; w2 < SMALL_WARPS; ++w2) s = radd(s, red[w2][bb]);
                    a.task_part[(int64_t)blockIdx.x * a.nblocks + bb] = s;
                }
            }
            grid.sync();
        }
        if (iter < a.max_iters) {
            // forces of slot A (hbcore.py:359-382): one warp per output, strict
            // left-to-right folds of the products h*q
            double *buf = fbuf[threadIdx.x >> 5];
            for (int t = gwarp; t < total_f; t += nwarps) {
                const int body = t % a.nbody;
                const int n = (t / a.nbody) % P;
                const int k = t / (a.nbody * P);
                double f = 0.0;
                for (int s = 0; s < a.nsegs; ++s) {
                    const hbgpu_force_seg g = a.segs[s];
                    if (g.body != body) continue;
                    const double *fp = a.slot[0] + g.start + (int64_t)(n * NPDE + k) * g.ps;
                    for (int c0 = 0; c0 < g.length; c0 += SMALL_FCH) {
#pragma unroll
                        for (int u = 0; u < SMALL_FCH / 32; ++u) {
                            const int c = c0 + lane + 32 * u;
                            buf[lane + 32 * u] = c < g.length ? rmul(g.h, fp[(int64_t)c * g.stride]) : 0.0;
                        }
                        __syncwarp();
                        if (lane == 0) {
                            const int m = min(SMALL_FCH, g.length - c0);
                            for (int e = 0; e < m; ++e) f = radd(f, buf[e]);
                        }
                        __syncwarp();
                    }
                }
                if (lane == 0) a.force_hist[(int64_t)iter * total_f + t] = f;
            }
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) *a.iter = a.it0 + a.iters;
}

struct SmallLaunch {
    void *fn = nullptr;
    int grid = 0;
    bool ready = false;
};

template <int P>
static int small_launch_p(const SmallArgs &a, int tasks, cudaStream_t s) {
    static SmallLaunch L_d[HB_MAX_DEVICES];
    const int dev = current_device();
    if (dev < 0) return HBGPU_ERR_CUDA;
    SmallLaunch &L = L_d[dev];
    if (!L.ready) {
        L.fn = (void *)small_kernel<P>;
        int sms = 0, per_sm = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, small_kernel<P>, SMALL_THREADS, 0) !=
                cudaSuccess ||
            per_sm < 1)
            return hbgpu_check_launch("small kernel occupancy");
        L.grid = sms * per_sm;
        L.ready = true;
    }
    // every co-resident CTA, or one warp per task if there are fewer tasks
    int grid = (int)std::min<int64_t>(L.grid, ((int64_t)tasks + SMALL_WARPS - 1) / SMALL_WARPS);
    grid = std::max(std::min(grid, SMALL_MAX_CTAS), 1);   // the partial buffer's capacity
    void *params[] = {(void *)&a};
    cudaError_t e = cudaLaunchCooperativeKernel(L.fn, dim3(grid), dim3(SMALL_THREADS), params, 0, s);
    if (e != cudaSuccess) {
        hbgpu_set_error("small kernel cooperative launch: %s", cudaGetErrorString(e));
        return HBGPU_ERR_CUDA;
    }
    hbgpu_count_launch(1);
    return HBGPU_OK;
}

// engine creation: the rank's warp-task count (from the device block table)
// and the per-task partial buffer
int small_prepare(const hbgpu_engine_desc &d, int *tasks, double **part_buf) {
    if (d.nblocks > SMALL_MAX_BLOCKS) {
        hbgpu_set_error("small schedule: %d blocks exceed %d", d.nblocks, SMALL_MAX_BLOCKS);
        return HBGPU_ERR_ARG;
    }
    std::vector<hbgpu_block> host(d.nblocks);
    if (cudaMemcpy(host.data(), d.blocks, sizeof(hbgpu_block) * d.nblocks, cudaMemcpyDeviceToHost) != cudaSuccess)
        return hbgpu_check_launch("small schedule: block table");
    int64_t n = 0;
    for (const hbgpu_block &b : host) n += (int64_t)((b.ni + 31) / 32) * NPDE * b.nj;
    if (n <= 0 || n > INT32_MAX / 2) {
        hbgpu_set_error("small schedule: %lld warp tasks", (long long)n);
        return HBGPU_ERR_ARG;
    }
    // one stage-0 partial per (CTA, block): at most one CTA per warp task
    const int64_t ctas = std::min<int64_t>((n + SMALL_WARPS - 1) / SMALL_WARPS, SMALL_MAX_CTAS);
    if (cudaMalloc(part_buf, sizeof(double) * (size_t)(ctas * d.nblocks)) != cudaSuccess)
        return hbgpu_check_launch("small schedule: partials");
    *tasks = (int)n;
    return HBGPU_OK;
}

// `iters` iterations of the engine described by `d` starting at iteration
// it0, in one cooperative launch (hb_runtime.cu, engine schedule "small")
int small_iterations(const hbgpu_engine_desc &d, int32_t it0, int32_t iters, cudaStream_t s, double *part_buf,
                     int tasks) {
    if (iters <= 0) return HBGPU_OK;
    SmallArgs a;
    memset(&a, 0, sizeof(a));
    for (int k = 0; k < 3; ++k) a.slot[k] = d.slot[k];
    a.blocks = d.blocks;
    a.sxy = d.sxy;
    a.faces = d.faces;
    a.status = d.status;
    a.iter = d.iter;
    a.sumsq = d.sumsq;
    a.segs = d.segs;
    a.force_hist = d.force_hist;
    a.nblocks = d.nblocks;
    a.planes = d.planes;
    a.nbody = d.nbody;
    a.nsegs = d.nsegs;
    a.it0 = it0;
    a.iters = iters;
    a.max_iters = d.max_iters;
    for (int k = 0; k < 4; ++k) a.coef[k] = d.coef[k];
    memcpy(a.D, d.D, sizeof(a.D));
    for (int k = 0; k < HBGPU_MAX_TEMPLATED_P * HBGPU_NPDE; ++k) a.ap[k] = d.ap[k];
    a.task_part = part_buf;
    switch (d.planes) {
        case 1: return small_launch_p<1>(a, tasks, s);
        case 3: return small_launch_p<3>(a, tasks, s);
        case 5: return small_launch_p<5>(a, tasks, s);
        case 7: return small_launch_p<7>(a, tasks, s);
        case 9: return small_launch_p<9>(a, tasks, s);
        default: break;
    }
    hbgpu_set_error("small schedule: P = %d not templated (1..9 odd)", d.planes);
    return HBGPU_ERR_UNSUPPORTED;
}

}  // namespace hbgpu
