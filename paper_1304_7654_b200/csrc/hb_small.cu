// hb_small.cu -- whole iterations of a small single-GPU rank in one launch.
//
// For a tiny rank (BASELINE C0: 2048 cells, 0.2 MB per slot) the per-stage
// TMA kernels spend most of their time in launch, pipeline fill and drain
// (7 launches per iteration, 28 us at C0).  Here one
// cooperative launch runs `iters` complete iterations: the 4 RK stages of
// every block (warps stride over (row, pde, 32-column chunk) tasks of each
// block; a thread computes one (cell, pde) for all P planes), separated by
// grid-wide barriers, with
//   * halo forwarding at write time through the face-target pool (local
//     cut halo cells of the output slot; the rank has no remote cuts),
//   * divergence keys per block (hbcore.py:279-284),
//   * stage 0: per-block sums of R^2 -- per thread in task order, per CTA in
//     a fixed tree, then over CTAs in order -- deterministic run to run,
//   * forces of each iteration into the history (CTA 0 after the last
//     stage; the next iteration's first stage only reads slot A),
// and the iteration counter set once at the end.  Operands come through L1
// and L2; every rounding is the reference's (strict rmul/radd, the signed
// zero terms included), so the fields equal the other schedules' bitwise.

#include "hb_tma.cuh"

#include <cooperative_groups.h>
#include <string.h>

#include <algorithm>

namespace cg = cooperative_groups;

namespace hbgpu {

constexpr int SMALL_THREADS = 128;
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
    double *cta_part;        // [nblocks * gridDim.x] stage-0 partials
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
__global__ void __launch_bounds__(SMALL_THREADS) small_kernel(const __grid_constant__ SmallArgs a) {
    cg::grid_group grid = cg::this_grid();
    __shared__ double red[SMALL_THREADS];
    const int lane = threadIdx.x & 31;
    const int nwarps = gridDim.x * (SMALL_THREADS / 32);
    const int gwarp = blockIdx.x * (SMALL_THREADS / 32) + (threadIdx.x >> 5);
    const int total_f = 3 * P * a.nbody;
    for (int it = 0; it < a.iters; ++it) {
        const int iter = a.it0 + it;
        for (int st = 0; st < 4; ++st) {
            const double *in = a.slot[in_slot_of(st)];
            const double *q0 = a.slot[0];
            double *out = a.slot[out_slot_of(st)];
            const int gstage = iter * 4 + st + 1;
            if (st == 1 && blockIdx.x == 0 && threadIdx.x < a.nblocks) {
                // this iteration's stage-0 partials, CTAs in order
                double s = 0.0;
                for (int c = 0; c < (int)gridDim.x; ++c) s = radd(s, a.cta_part[threadIdx.x * gridDim.x + c]);
                a.sumsq[(int64_t)iter * a.nblocks + threadIdx.x] = s;
            }
            for (int bidx = 0; bidx < a.nblocks; ++bidx) {
                const hbgpu_block b = a.blocks[bidx];
                // warp tasks: (row j, pde p, 32-column chunk), chunk fastest
                const int chunks = (b.ni + 31) >> 5;
                const int tasks = chunks * NPDE * b.nj;
                double acc = 0.0;
                for (int t = gwarp; t < tasks; t += nwarps) {
                    const int chunk = t % chunks;
                    const int r = t / chunks;
                    const int p = r % NPDE, j = r / NPDE + 1;
                    const int i = (chunk << 5) + lane + 1;
                    if (i <= b.ni) acc += small_cell<P>(a, b, in, q0, out, st, p, j, i, gstage, bidx);
                }
                if (st == 0) {
                    // fixed-shape tree over the CTA's threads
                    red[threadIdx.x] = acc;
                    __syncthreads();
                    for (int w = SMALL_THREADS / 2; w > 0; w >>= 1) {
                        if (threadIdx.x < w) red[threadIdx.x] = radd(red[threadIdx.x], red[threadIdx.x + w]);
                        __syncthreads();
                    }
                    if (threadIdx.x == 0) a.cta_part[bidx * gridDim.x + blockIdx.x] = red[0];
                    __syncthreads();
                }
            }
            grid.sync();
        }
        if (blockIdx.x == 0 && iter < a.max_iters) {
            // forces of slot A (hbcore.py:359-382), strict left-to-right folds
            for (int t = threadIdx.x; t < total_f; t += blockDim.x) {
                const int body = t % a.nbody;
                const int n = (t / a.nbody) % P;
                const int k = t / (a.nbody * P);
                double f = 0.0;
                for (int s = 0; s < a.nsegs; ++s) {
                    const hbgpu_force_seg g = a.segs[s];
                    if (g.body != body) continue;
                    const double *fp = a.slot[0] + g.start + (int64_t)(n * NPDE + k) * g.ps;
                    for (int c = 0; c < g.length; ++c) f = radd(f, rmul(g.h, fp[(int64_t)c * g.stride]));
                }
                a.force_hist[(int64_t)iter * total_f + t] = f;
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
static int small_launch_p(const SmallArgs &args, int64_t max_items, cudaStream_t s, double **part_buf,
                          int *part_cap) {
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
    // one warp task per (row, pde, 32 columns) of the largest block
    int grid = (int)std::min<int64_t>(L.grid, (max_items / P + SMALL_THREADS - 1) / SMALL_THREADS);
    grid = std::max(grid, 1);
    SmallArgs a = args;
    const int need = a.nblocks * grid;
    if (*part_cap < need) {
        if (*part_buf) cudaFree(*part_buf);
        *part_buf = nullptr;
        *part_cap = 0;
        if (cudaMalloc(part_buf, sizeof(double) * (size_t)need) != cudaSuccess)
            return hbgpu_check_launch("small kernel partials");
        *part_cap = need;
    }
    a.cta_part = *part_buf;
    void *params[] = {(void *)&a};
    cudaError_t e = cudaLaunchCooperativeKernel(L.fn, dim3(grid), dim3(SMALL_THREADS), params, 0, s);
    if (e != cudaSuccess) {
        hbgpu_set_error("small kernel cooperative launch: %s", cudaGetErrorString(e));
        return HBGPU_ERR_CUDA;
    }
    hbgpu_count_launch(1);
    return HBGPU_OK;
}

// `iters` iterations of the engine described by `d` starting at iteration
// it0, in one cooperative launch (hb_runtime.cu, engine schedule "small")
int small_iterations(const hbgpu_engine_desc &d, int32_t it0, int32_t iters, cudaStream_t s, double **part_buf,
                     int *part_cap) {
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
    const int64_t max_items = (int64_t)d.planes * NPDE * (int64_t)d.small_max_cells;
    switch (d.planes) {
        case 1: return small_launch_p<1>(a, max_items, s, part_buf, part_cap);
        case 3: return small_launch_p<3>(a, max_items, s, part_buf, part_cap);
        case 5: return small_launch_p<5>(a, max_items, s, part_buf, part_cap);
        case 7: return small_launch_p<7>(a, max_items, s, part_buf, part_cap);
        case 9: return small_launch_p<9>(a, max_items, s, part_buf, part_cap);
        default: break;
    }
    hbgpu_set_error("small schedule: P = %d not templated (1..9 odd)", d.planes);
    return HBGPU_ERR_UNSUPPORTED;
}

}  // namespace hbgpu
