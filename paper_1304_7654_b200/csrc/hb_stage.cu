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
//   * stage 0: per-CTA partial sums of R^2 for the residual norm.
//
// Layout and mapping.  A CTA is 4 warps; warp w owns pde p = w and 32
// consecutive interior columns i; every lane marches down `tile_rows` rows
// j keeping the rows j-1, j, j+1 of all P snapshots of its column in
// registers (the stencil's north/south neighbours and the P centres the
// D-contraction needs).  West/east neighbours come from the adjacent lanes
// by warp shuffle; only lanes 0 and 31 load them.  Each q value therefore
// crosses HBM once per stage (plus two halo rows per tile), and a warp's
// loads and stores are 256 B contiguous rows.
//
// Rounding: every operation is an explicitly rounded DMUL/DADD, in the
// reference's per-point order, including the m == n term (D[n][n] = 0 still
// contributes a signed zero) and the +ap*sxy term on zero-amplitude planes.

#include "hb_common.cuh"

namespace hbgpu {

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

__device__ __forceinline__ void forward(const FaceHit &t, double *out, double *sendbuf, int n, int p,
                                        double v) {
    if (t.ps > 0) {
        out[t.off + (int64_t)(n * NPDE + p) * t.ps] = v;
    } else if (t.ps < 0) {
        sendbuf[t.off + n * NPDE + p] = v;
    }
}

__device__ __forceinline__ double cta_sum(double v, double *smem) {
    // fixed-shape tree: deterministic for a given launch geometry
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = radd(v, __shfl_down_sync(0xffffffffu, v, o));
    const int warp = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) smem[warp] = v;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x == 0) {
        s = smem[0];
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) s = radd(s, smem[w]);
    }
    return s;
}

template <int P, bool FIRST>
__global__ void __launch_bounds__(128) stage_kernel(const __grid_constant__ hbgpu_stage_args a) {
    __shared__ double red[4];
    const int cta = blockIdx.x;
    const int bidx = a.cta_block[cta];
    const hbgpu_block &blk = a.blocks[bidx];
    const int ni = blk.ni, nj = blk.nj, pitch = blk.pitch;
    const int64_t ps = blk.ps;
    const int64_t ps4 = ps * NPDE;
    const double nu_h2 = blk.nu_h2, adv_2h = blk.adv_2h;

    const int local = cta - blk.cta_begin;
    const int ti = local % blk.tiles_i;
    const int tj = local / blk.tiles_i;
    const int lane = threadIdx.x & 31;
    const int p = threadIdx.x >> 5;
    const int i = ti * 32 + lane + 1;            // 1-based interior column
    const bool live = i <= ni;
    const int ic = min(i, ni + 1);               // clamped: dead lanes read the halo column
    const int j0 = tj * a.tile_rows + 1;
    const int j1 = min(j0 + a.tile_rows - 1, nj);
    const int gstage = (*a.iter) * 4 + a.stage + 1;

    const int64_t col = blk.base + (int64_t)p * ps + LEAD + ic;
    const double *__restrict__ in = a.in + col;
    const double *q0 = a.q0 + col;
    double *out = a.out + col;
    const double *sxy = a.sxy + blk.sxy_off + (i - 1);
    const double coef = a.coef;

    double up[P], cur[P], dn[P];
#pragma unroll
    for (int m = 0; m < P; ++m) {
        up[m] = __ldg(in + m * ps4 + (int64_t)(j0 - 1) * pitch);
        cur[m] = __ldg(in + m * ps4 + (int64_t)j0 * pitch);
    }

    double nrm = 0.0;
    // west/east neighbours outside the warp's 32 columns
    const int64_t wcol = (int64_t)(i - 1) - ic;                 // offset of column i-1
    const int64_t ecol = (int64_t)min(i + 1, ni + 1) - ic;      // offset of column i+1

    for (int j = j0; j <= j1; ++j) {
        const int64_t row = (int64_t)j * pitch;
#pragma unroll
        for (int m = 0; m < P; ++m) dn[m] = __ldg(in + m * ps4 + row + pitch);
        double q0v[FIRST ? 1 : P];
        if (!FIRST) {
#pragma unroll
            for (int n = 0; n < P; ++n) q0v[n] = q0[n * ps4 + row];
        }
        const double sv = live ? sxy[(int64_t)(j - 1) * ni] : 0.0;

        FaceHit trow{0, 0}, tcol{0, 0};
        if (live) {
            if (j == 1) trow = load_target(a.faces, blk.face_off[0], i - 1);
            else if (j == nj) trow = load_target(a.faces, blk.face_off[1], i - 1);
            if (i == 1) tcol = load_target(a.faces, blk.face_off[2], j - 1);
            else if (i == ni) tcol = load_target(a.faces, blk.face_off[3], j - 1);
        }

#pragma unroll
        for (int n = 0; n < P; ++n) {
            const double *rown = in + n * ps4 + row;
            double w = __shfl_up_sync(0xffffffffu, cur[n], 1);
            double e = __shfl_down_sync(0xffffffffu, cur[n], 1);
            if (lane == 0) w = __ldg(rown + wcol);
            if (lane == 31) e = __ldg(rown + ecol);
            double o = stencil(cur[n], w, e, up[n], dn[n], nu_h2, adv_2h);
#pragma unroll
            for (int m = 0; m < P; ++m) o = radd(o, rmul(a.D[n * P + m], cur[m]));
            o = radd(o, rmul(a.ap[n * NPDE + p], sv));
            const double base = FIRST ? cur[n] : q0v[n];
            const double v = rsub(base, rmul(coef, o));
            if (live) {
                out[n * ps4 + row] = v;
                if (FIRST) nrm = radd(nrm, rmul(o, o));
                forward(trow, a.out, a.sendbuf, n, p, v);
                forward(tcol, a.out, a.sendbuf, n, p, v);
                if (nonfinite(v)) {
                    long long lin = (((long long)(n * NPDE + p) * nj + (j - 1)) * ni) + (i - 1);
                    atomicMin(a.status + bidx, divergence_key(gstage, lin));
                }
            }
        }
#pragma unroll
        for (int m = 0; m < P; ++m) {
            up[m] = cur[m];
            cur[m] = dn[m];
        }
    }
    if (FIRST && a.norm_part != nullptr) {
        double s = cta_sum(nrm, red);
        if (threadIdx.x == 0) a.norm_part[cta] = s;
    }
}

// Generic snapshot count (P > HBGPU_MAX_TEMPLATED_P, e.g. the 63-plane
// tc1-full case): one thread per (column, pde) and row, D from shared memory,
// operands re-read through L1.  Same arithmetic sequence.
__global__ void __launch_bounds__(128) stage_kernel_generic(const __grid_constant__ hbgpu_stage_args a) {
    extern __shared__ double sh[];
    double *D = sh;
    double *red = sh + a.planes * a.planes;
    const int P = a.planes;
    for (int k = threadIdx.x; k < P * P; k += blockDim.x) D[k] = a.dmat[k];
    __syncthreads();
    const int cta = blockIdx.x;
    const int bidx = a.cta_block[cta];
    const hbgpu_block &blk = a.blocks[bidx];
    const int ni = blk.ni, nj = blk.nj, pitch = blk.pitch;
    const int64_t ps4 = blk.ps * NPDE;
    const int local = cta - blk.cta_begin;
    const int ti = local % blk.tiles_i, tj = local / blk.tiles_i;
    const int lane = threadIdx.x & 31, p = threadIdx.x >> 5;
    const int i = ti * 32 + lane + 1;
    const bool live = i <= ni;
    const int j0 = tj * a.tile_rows + 1, j1 = min(j0 + a.tile_rows - 1, nj);
    const bool first = a.stage == 0;
    const int gstage = (*a.iter) * 4 + a.stage + 1;
    double nrm = 0.0;
    if (live) {
        const int64_t col = blk.base + (int64_t)blk.ps * p + LEAD + i;
        const double *in = a.in + col;
        for (int j = j0; j <= j1; ++j) {
            const int64_t row = (int64_t)j * pitch;
            const double sv = a.sxy[blk.sxy_off + (int64_t)(j - 1) * ni + (i - 1)];
            FaceHit trow{0, 0}, tcol{0, 0};
            if (j == 1) trow = load_target(a.faces, blk.face_off[0], i - 1);
            else if (j == nj) trow = load_target(a.faces, blk.face_off[1], i - 1);
            if (i == 1) tcol = load_target(a.faces, blk.face_off[2], j - 1);
            else if (i == ni) tcol = load_target(a.faces, blk.face_off[3], j - 1);
            for (int n = 0; n < P; ++n) {
                const double *c = in + n * ps4 + row;
                double o = stencil(c[0], c[-1], c[1], c[-pitch], c[pitch], blk.nu_h2, blk.adv_2h);
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
                    atomicMin(a.status + bidx, divergence_key(gstage, lin));
                }
            }
        }
    }
    if (first && a.norm_part != nullptr) {
        double s = cta_sum(nrm, red);
        if (threadIdx.x == 0) a.norm_part[cta] = s;
    }
}

template <int P>
static void launch_p(const hbgpu_stage_args &a, cudaStream_t s) {
    if (a.stage == 0)
        stage_kernel<P, true><<<a.total_ctas, 128, 0, s>>>(a);
    else
        stage_kernel<P, false><<<a.total_ctas, 128, 0, s>>>(a);
}

}  // namespace hbgpu

extern "C" int hbgpu_stage(const hbgpu_stage_args *args, void *stream) {
    using namespace hbgpu;
    if (args == nullptr || args->total_ctas <= 0 || args->planes < 1) {
        hbgpu_set_error("hbgpu_stage: bad arguments");
        return HBGPU_ERR_ARG;
    }
    cudaStream_t s = (cudaStream_t)stream;
    const hbgpu_stage_args &a = *args;
    switch (a.planes) {
        case 1: launch_p<1>(a, s); break;
        case 3: launch_p<3>(a, s); break;
        case 5: launch_p<5>(a, s); break;
        case 7: launch_p<7>(a, s); break;
        case 9: launch_p<9>(a, s); break;
        case 11: launch_p<11>(a, s); break;
        case 13: launch_p<13>(a, s); break;
        case 15: launch_p<15>(a, s); break;
        case 17: launch_p<17>(a, s); break;
        default: {
            if (a.dmat == nullptr) {
                hbgpu_set_error("hbgpu_stage: P=%d needs args->dmat", a.planes);
                return HBGPU_ERR_ARG;
            }
            size_t sm = sizeof(double) * ((size_t)a.planes * a.planes + 4);
            if (sm > 48 * 1024)
                cudaFuncSetAttribute(stage_kernel_generic, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)sm);
            stage_kernel_generic<<<a.total_ctas, 128, sm, s>>>(a);
        }
    }
    hbgpu_count_launch(1);
    return hbgpu_check_launch("hbgpu_stage");
}
