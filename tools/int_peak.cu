// int_peak.cu — achievable integer issue rate of the B200: every SM runs warps of
// independent IADD3 / LOP3 chains (8 accumulators per thread, no memory traffic in the loop), timed with CUDA
// events. Reports lane-ops/s = threads x iterations x ops per iteration / seconds, the denominator of the
// "alu" roofline in bench.py when profiles/int_peak.json exists.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o int_peak tools/int_peak.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

// MIX = 0: IADD3 + LOP3 (alu pipe only); MIX = 1: half the ops are IMAD (fma pipe), interleaved with alu-pipe ops.
template <int MIX>
__global__ void __launch_bounds__(256) k_int(uint32_t iters, uint32_t seed, uint32_t* out) {
    uint32_t a0 = threadIdx.x ^ seed, a1 = a0 * 3u, a2 = a0 * 5u, a3 = a0 * 7u, a4 = a0 * 11u, a5 = a0 * 13u,
             a6 = a0 * 17u, a7 = a0 * 19u;
    const uint32_t k = seed | 1u;
#pragma unroll 1
    for (uint32_t i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {  // 16 integer ops per unrolled step: 8 IADD3 + 8 LOP3, 8 independent chains
            a0 = a0 + a1 + k;
            a1 = a1 + a2 + k;
            a2 = a2 + a3 + k;
            a3 = a3 + a4 + k;
            a4 = a4 + a5 + k;
            a5 = a5 + a6 + k;
            a6 = a6 + a7 + k;
            a7 = a7 + a0 + k;
            if (MIX) {  // IMAD: a*k + b on the fma pipe
                a0 = a0 * k + a1;
                a1 = a1 * k + a2;
                a2 = a2 * k + a3;
                a3 = a3 * k + a4;
                a4 = a4 * k + a5;
                a5 = a5 * k + a6;
                a6 = a6 * k + a7;
                a7 = a7 * k + a0;
            } else {
                a0 = (a0 & a1) ^ a2;
                a1 = (a1 | a2) ^ a3;
                a2 = (a2 & a3) ^ a4;
                a3 = (a3 | a4) ^ a5;
                a4 = (a4 & a5) ^ a6;
                a5 = (a5 | a6) ^ a7;
                a6 = (a6 & a7) ^ a0;
                a7 = (a7 | a0) ^ a1;
            }
        }
    }
    const uint32_t r = a0 ^ a1 ^ a2 ^ a3 ^ a4 ^ a5 ^ a6 ^ a7;
    if (r == 0x12345678u) out[blockIdx.x] = r;  // keep the chains live
}

template <int MIX>
static double run(int sms, uint32_t* out, int* per_sm_out) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_int<MIX>, 256, 0);
    *per_sm_out = per_sm;
    const uint32_t blocks = (uint32_t)(sms * per_sm), iters = 20000;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    k_int<MIX><<<blocks, 256>>>(iters / 10, 7u, out);  // warm-up (clocks)
    cudaDeviceSynchronize();
    double best = 0;
    for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(a);
        k_int<MIX><<<blocks, 256>>>(iters, 7u + rep, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        const double rate = (double)blocks * 256 * iters * 4 * 16 / (ms * 1e-3);
        if (rate > best) best = rate;
    }
    return best;
}

int main() {
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    uint32_t* out;
    cudaMalloc(&out, 65536 * 4);
    const double alu = run<0>(sms, out, &per_sm);
    const double mix = run<1>(sms, out, &per_sm);
    printf("{\"int_lane_ops_per_s\": %.6e, \"alu_only_lane_ops_per_s\": %.6e, \"alu_fma_mix_lane_ops_per_s\": %.6e, "
           "\"sms\": %d, \"blocks_per_sm\": %d, \"threads_per_block\": 256, \"ops\": \"8 independent 32-bit chains per "
           "thread: IADD3 + LOP3 (alu pipe), or IADD3 + IMAD (alu + fma pipes)\"}\n",
           alu > mix ? alu : mix, alu, mix, sms, per_sm);
    return 0;
}
