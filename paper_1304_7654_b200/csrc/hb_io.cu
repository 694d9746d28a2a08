// hb_io.cu -- restart / flowtec records packed on the device.
//
// The reference writes its output files record by record from host arrays
// (outio.py:107-123 record_payload, 221-241 write_records): per (block,
// plane) a 4-byte length prefix, the float64 payload in (row, column,
// variable) order, and the same 4-byte suffix, records dense in the file.
// Here the interior of a slot is transposed into that byte image directly on
// the device, so the host only moves finished bytes (one D2H copy and one
// positioned write per run of records).  Records start at 4-byte offsets, so
// every double is stored as two 32-bit words; a warp writes 32 consecutive
// cells = 1 KB contiguous.

#include "hb_common.cuh"

namespace hbgpu {

__global__ void pack_records_kernel(const double *slot, const hbgpu_block *blocks, const hbgpu_out_record *recs,
                                    const double *xy, uint32_t *dst) {
    const hbgpu_out_record r = recs[blockIdx.y];
    const hbgpu_block b = blocks[r.block];
    const int64_t cells = (int64_t)b.ni * b.nj;
    const uint32_t payload = (uint32_t)(cells * 4 * sizeof(double));
    uint32_t *rec = dst + r.dst / 4;   // r.dst is a multiple of 4
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        rec[0] = payload;
        rec[1 + payload / 4] = payload;
    }
    uint32_t *body = rec + 1;
    const double *plane = slot + b.base + (int64_t)r.plane * NPDE * b.ps + HBGPU_ROW_LEAD;
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < cells; c += (int64_t)gridDim.x * blockDim.x) {
        const int j = (int)(c / b.ni) + 1;
        const int i = (int)(c - (int64_t)(j - 1) * b.ni) + 1;
        const double *cell = plane + (int64_t)j * b.rs + i;
        double v[4];
        if (r.kind == HBGPU_RECORD_RESTART) {
#pragma unroll
            for (int p = 0; p < NPDE; ++p) v[p] = cell[p * b.ps];
        } else {
            v[0] = xy[r.xy + i - 1];
            v[1] = xy[r.xy + b.ni + j - 1];
            v[2] = cell[0];
            v[3] = cell[b.ps];
        }
        uint32_t *out = body + c * 8;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const unsigned long long bits = (unsigned long long)__double_as_longlong(v[k]);
            out[2 * k] = (uint32_t)bits;             // little-endian: low word first
            out[2 * k + 1] = (uint32_t)(bits >> 32);
        }
    }
}

}  // namespace hbgpu

extern "C" int hbgpu_pack_records(const double *slot, const hbgpu_block *blocks, const hbgpu_out_record *recs,
                                  int32_t nrecs, int32_t max_cells, const double *xy, void *dst, void *stream) {
    if (nrecs < 0 || nrecs > 65535 || max_cells < 0 || (nrecs > 0 && (slot == nullptr || blocks == nullptr ||
                                                                        recs == nullptr || dst == nullptr))) {
        hbgpu_set_error("hbgpu_pack_records: bad arguments (nrecs %d, max_cells %d)", nrecs, max_cells);
        return HBGPU_ERR_ARG;
    }
    if (((uintptr_t)dst & 3) != 0) {
        hbgpu_set_error("hbgpu_pack_records: dst must be 4-byte aligned");
        return HBGPU_ERR_ARG;
    }
    if (nrecs == 0) return HBGPU_OK;
    const int threads = 256;
    const int64_t want = ((int64_t)max_cells + threads - 1) / threads;
    const dim3 grid((unsigned)(want < 1 ? 1 : (want > 1024 ? 1024 : want)), (unsigned)nrecs);
    hbgpu::pack_records_kernel<<<grid, threads, 0, (cudaStream_t)stream>>>(slot, blocks, recs, xy, (uint32_t *)dst);
    hbgpu_count_launch(1);
    return hbgpu_check_launch("hbgpu_pack_records");
}
