// fp64_peak.cu -- measured fp64 arithmetic throughput of this B200, the
// compute roofline of the paired-stage kernel (which issues separately
// rounded DMUL / DADD, no FMA: the reference's rounding).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
//   ./fp64_peak   ->  one JSON line: DADD, DMUL and DFMA instruction rates
//
// Each thread runs 16 independent dependency chains of 4096 operations; the
// grid is 148 SMs x 8 CTAs x 256 threads.  Rates are warp-lane operations
// per second (an FMA counts as one instruction, two flops).
#include <cstdio>
#include <cuda_runtime.h>

constexpr int CHAINS = 16, ITERS = 4096;

template <int OP>
__global__ void spin(double *out, double x, double y) {
    double a[CHAINS];
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) a[c] = x + c * 1e-3 + threadIdx.x * 1e-9;
    for (int k = 0; k < ITERS; ++k) {
#pragma unroll
        for (int c = 0; c < CHAINS; ++c) {
            if (OP == 0) a[c] = __dadd_rn(a[c], y);
            else if (OP == 1) a[c] = __dmul_rn(a[c], y);
            else a[c] = __fma_rn(a[c], y, x);
        }
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) s += a[c];
    if (s == 12345.678) out[0] = s;   // keep the chains alive
}

template <int OP>
static double rate(int sms) {
    double *out;
    cudaMalloc(&out, 8);
    dim3 grid(sms * 8), block(256);
    spin<OP><<<grid, block>>>(out, 1.0, 0.999999);
    cudaDeviceSynchronize();
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) spin<OP><<<grid, block>>>(out, 1.0, 0.999999);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    cudaFree(out);
    return 5.0 * grid.x * block.x * (double)CHAINS * ITERS / (ms * 1e-3);
}

int main() {
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const double dadd = rate<0>(sms), dmul = rate<1>(sms), dfma = rate<2>(sms);
    printf("{\"dadd_ops_per_s\": %.4e, \"dmul_ops_per_s\": %.4e, \"dfma_ops_per_s\": %.4e, "
           "\"sms\": %d, \"max_clock_khz\": %d, \"lanes_per_sm_per_clk_at_max\": %.1f}\n",
           dadd, dmul, dfma, sms, clk, dadd / (sms * (clk * 1e3)));
    return 0;
}
