// libtracegen.so — host and device entry points of the seeded trace generator (input generation only; see
// tracegen.h). Used by tests (host traces for the oracle), by bench.py (device-resident traces; pinned host traces
// for the end-to-end leg) and by smoke(). Holds none of the method's arithmetic.
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include "tracegen.h"

extern "C" {

uint32_t tg_cfg_jobs_per_trace(uint32_t cfg) { return tg_jobs_per_trace(cfg); }
uint32_t tg_cfg_has_ext(uint32_t cfg) { return tg_has_ext(cfg); }
uint64_t tg_cfg_seed(uint32_t cfg) { return TG_SEED(cfg); }

// Host generation of traces [trace_id0, trace_id0 + n) into caller arrays: jobs (n*J*4 u32), ext (n*J*4 u32 or
// NULL), trace_off (n+1 u64, local offsets starting at 0). Returns 0, or -1 for an unknown cfg.
int tg_generate_host(uint32_t cfg, uint64_t seed, uint64_t trace_id0, uint64_t n, uint32_t* jobs, uint32_t* ext,
                     uint64_t* trace_off) {
    const uint32_t J = tg_jobs_per_trace(cfg);
    if (J == 0) return -1;
#pragma omp parallel for schedule(static)
    for (int64_t t = 0; t < (int64_t)n; ++t) {
        uint32_t* je = ext ? ext + (uint64_t)t * J * 4 : nullptr;
        if (ext) memset(je, 0, sizeof(uint32_t) * 4 * J);
        tg_gen_trace(cfg, seed, trace_id0 + (uint64_t)t, jobs + (uint64_t)t * J * 4, je);
    }
    if (trace_off)
        for (uint64_t t = 0; t <= n; ++t) trace_off[t] = t * J;
    return 0;
}

// Dynamic-job samples y[1..T], q[1..T] (written to y[0..T-1], q[0..T-1]) for one job record (tests only).
void tg_dyn_samples_host(uint64_t seed, uint64_t trace_id, uint32_t job_idx, const uint32_t* job, const uint32_t* ext,
                         uint32_t T, uint32_t* y, uint32_t* q) {
    uint64_t key = tg_key(seed, trace_id, job_idx);
    for (uint32_t i = 1; i <= T; ++i)
        tg_dyn_sample(key, i, job[0], ext[2], ext[3] & 0xFFFFu, job[1], ext[3] >> 16, &y[i - 1], &q[i - 1]);
}

// The same through tg_dyn_sample_fast (tests: equality under its range bounds).
void tg_dyn_samples_host_fast(uint64_t seed, uint64_t trace_id, uint32_t job_idx, const uint32_t* job,
                              const uint32_t* ext, uint32_t T, uint32_t* y, uint32_t* q) {
    uint64_t key = tg_key(seed, trace_id, job_idx);
    for (uint32_t i = 1; i <= T; ++i)
        tg_dyn_sample_fast(key, i, job[0], ext[2], ext[3] & 0xFFFFu, job[1], ext[3] >> 16, &y[i - 1], &q[i - 1]);
}

}  // extern "C"

__global__ void tg_generate_kernel(uint32_t cfg, uint64_t seed, uint64_t trace_id0, uint64_t n, uint32_t J,
                                   uint4* __restrict__ jobs, uint4* __restrict__ ext, uint64_t* __restrict__ off) {
    uint32_t lj[4 * TG_MAX_JOBS_PER_TRACE];
    uint32_t le[4 * TG_MAX_JOBS_PER_TRACE];
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < n; t += (uint64_t)gridDim.x * blockDim.x) {
        for (uint32_t k = 0; k < 4 * J; ++k) le[k] = 0;
        tg_gen_trace(cfg, seed, trace_id0 + t, lj, ext ? le : nullptr);
        for (uint32_t j = 0; j < J; ++j) {
            jobs[t * J + j] = make_uint4(lj[4 * j], lj[4 * j + 1], lj[4 * j + 2], lj[4 * j + 3]);
            if (ext) ext[t * J + j] = make_uint4(le[4 * j], le[4 * j + 1], le[4 * j + 2], le[4 * j + 3]);
        }
        off[t] = t * J;
        if (t == n - 1) off[n] = n * J;
    }
}

extern "C" int tg_generate_device(uint32_t cfg, uint64_t seed, uint64_t trace_id0, uint64_t n, void* jobs, void* ext,
                                  void* trace_off, void* stream) {
    const uint32_t J = tg_jobs_per_trace(cfg);
    if (J == 0) return -1;
    if (n == 0) return 0;
    int threads = 128;
    uint64_t blocks = (n + threads - 1) / threads;
    if (blocks > 148 * 64) blocks = 148 * 64;
    tg_generate_kernel<<<(unsigned)blocks, threads, 0, (cudaStream_t)stream>>>(
        cfg, seed, trace_id0, n, J, (uint4*)jobs, (uint4*)ext, (uint64_t*)trace_off);
    return cudaGetLastError() == cudaSuccess ? 0 : -2;
}
