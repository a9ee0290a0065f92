// trace_order.cu — the order in which the lane kernels visit a call's traces (a scheduling choice of the engine, not
// part of the method: every trace's result and every per-policy total is the same in any order).
//
// A lane simulates one trace at a time and a warp executes the union of its 32 lanes' paths each loop iteration
// (simulate_ff.cu, simulate_lane.cu). Traces whose queues start alike (the same tight-fit levels for their first
// jobs, the same iteration time: the paper's homogeneous mixes) step through the same sequence of events
// and decisions, so when the lanes of a warp hold such traces they take the same paths in the same iterations. The
// pass below bins the traces by that signature (a counting sort over at most 8192 keys) and the lane kernels take
// their units through the resulting permutation: config 2's FUSION_FISSION launch 2.85 -> 2.5 ms.
#include <algorithm>

#include "lane_common.cuh"

namespace mig {

constexpr uint32_t kOrderKeys = 8192;  // 1 same-iteration-time bit + 4 jobs x 3-bit tight-fit level
constexpr uint32_t kOrderJobs = 4;

struct OrderParams {
    const uint4* jobs;
    const uint4* ext;
    const uint64_t* off;
    uint64_t n_traces;
    uint32_t level_mem[kMaxLevels];
    uint32_t n_levels, mem0, ctx;
};

// Signature of a trace: the tight-fit level of each of its first kOrderJobs jobs (est + ws + ctx; a DYNAMIC job starts
// on the smallest slice, R16; 7 = no such job) and whether their iteration times agree.
__device__ __forceinline__ uint32_t trace_key(const OrderParams& P, uint64_t t) {
    const uint64_t o0 = P.off[t], o1 = P.off[t + 1], j0 = o0 - P.off[0];
    const uint32_t n = o1 - o0 < kOrderJobs ? (uint32_t)(o1 - o0) : kOrderJobs;
    uint32_t key = 0, same = 1, w0 = 0;
    for (uint32_t k = 0; k < kOrderJobs; ++k) {
        uint32_t lev = 7;
        if (k < n) {
            const uint4 r = __ldg(P.jobs + j0 + k);
            const uint32_t ws = P.ext ? __ldg(&P.ext[j0 + k].x) : 0u;
            const uint32_t req = ((r.z >> 16) & 0xFFu) == kClassDynamic ? P.mem0 : r.x + ws + P.ctx;
            lev = 0;
            for (uint32_t l = 0; l < P.n_levels; ++l) lev += P.level_mem[l] < req ? 1u : 0u;
            if (k == 0) w0 = r.w;
            same &= r.w == w0 ? 1u : 0u;
        }
        key = key * 8 + lev;
    }
    return (same << 12) | key;
}

// Pass 1: each trace's key, and the key histogram (per-CTA in shared memory, then one atomic per used bin).
__global__ void __launch_bounds__(256) k_order_keys(const OrderParams P, uint16_t* keys, uint32_t* hist) {
    __shared__ uint32_t h[kOrderKeys];
    for (uint32_t i = threadIdx.x; i < kOrderKeys; i += blockDim.x) h[i] = 0;
    __syncthreads();
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < P.n_traces;
         t += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t key = trace_key(P, t);
        keys[t] = (uint16_t)key;
        atomicAdd(h + key, 1u);
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < kOrderKeys; i += blockDim.x)
        if (h[i]) atomicAdd(hist + i, h[i]);
}

// Pass 2: exclusive prefix sum of the histogram, in place (one CTA of 1024 threads, 8 bins each). hist[kOrderKeys]
// (one word past the bins) receives the decision: 1 = order by key, 0 = keep trace order, when fewer than a quarter of
// the traces start with jobs of one iteration time (the homogeneous queues whose lanes fall into step; a call of
// mixed queues gains no phase alignment and would only lose the record locality of trace order).
__global__ void __launch_bounds__(1024) k_order_scan(uint32_t* hist, uint64_t n, bool force) {
    __shared__ uint32_t part[1024];
    __shared__ unsigned long long same;
    const uint32_t tid = threadIdx.x;
    if (tid == 0) same = 0;
    __syncthreads();
    if (tid >= 512) {  // keys with the same-iteration-time bit (bit 12) are bins 4096..8191
        uint32_t c = 0;
#pragma unroll
        for (int k = 0; k < 8; ++k) c += hist[tid * 8 + k];
        atomicAdd(&same, (unsigned long long)c);
    }
    uint32_t v[8], s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        v[k] = hist[tid * 8 + k];
        s += v[k];
    }
    part[tid] = s;
    __syncthreads();
    for (uint32_t d = 1; d < 1024; d <<= 1) {  // inclusive scan of the per-thread sums
        const uint32_t x = tid >= d ? part[tid - d] : 0u;
        __syncthreads();
        part[tid] += x;
        __syncthreads();
    }
    uint32_t run = part[tid] - s;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        hist[tid * 8 + k] = run;
        run += v[k];
    }
    if (tid == 0) hist[kOrderKeys] = force || 4 * same >= n ? 1u : 0u;
}

// Pass 3: scatter the trace ids to their bins. Each CTA takes a contiguous range of traces, counts its keys in
// shared memory, reserves its share of every bin it uses with one global atomic, and places its traces with shared
// atomics (a hot bin is then touched once per CTA in global memory, not once per warp). The order inside a bin is
// whatever the atomics give, which only changes the schedule.
__global__ void __launch_bounds__(256) k_order_scatter(const uint16_t* keys, uint32_t* cursor, uint32_t* order,
                                                      uint64_t n) {
    if (!cursor[kOrderKeys]) {  // keep trace order (k_order_scan's decision)
        for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < n; t += (uint64_t)gridDim.x * blockDim.x)
            order[t] = (uint32_t)t;
        return;
    }
    __shared__ uint32_t h[kOrderKeys];
    for (uint32_t i = threadIdx.x; i < kOrderKeys; i += blockDim.x) h[i] = 0;
    __syncthreads();
    const uint64_t per = (n + gridDim.x - 1) / gridDim.x, t0 = blockIdx.x * per, t1 = min(n, t0 + per);
    for (uint64_t t = t0 + threadIdx.x; t < t1; t += blockDim.x) atomicAdd(h + keys[t], 1u);
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < kOrderKeys; i += blockDim.x)
        if (h[i]) h[i] = atomicAdd(cursor + i, h[i]);
    __syncthreads();
    for (uint64_t t = t0 + threadIdx.x; t < t1; t += blockDim.x) order[atomicAdd(h + keys[t], 1u)] = (uint32_t)t;
}

size_t trace_order_scratch_bytes(uint64_t n_traces) {
    return ((n_traces * 4 + 255) & ~(size_t)255) + ((n_traces * 2 + 255) & ~(size_t)255) + (kOrderKeys + 1) * 4;
}

// buf: trace_order_scratch_bytes(n_traces) of scratch; the visit order (n_traces u32) is written at its start, the
// keys and the histogram follow. force: order by key whatever the share of homogeneous queues. Three launches.
cudaError_t launch_trace_order(const mig_traces& tr, const DevGeom* Gh, uint32_t ctx, void* buf, bool force,
                               int sm_count, cudaStream_t s) {
    OrderParams P;
    P.jobs = (const uint4*)tr.jobs;
    P.ext = (const uint4*)tr.jobs_ext;
    P.off = tr.trace_off;
    P.n_traces = tr.n_traces;
    P.n_levels = Gh->n_levels;
    for (int l = 0; l < kMaxLevels; ++l) P.level_mem[l] = l < (int)Gh->n_levels ? Gh->level_mem[l] : 0xFFFFFFFFu;
    P.mem0 = Gh->mem[0];
    P.ctx = ctx;
    char* sc = static_cast<char*>(buf);
    uint32_t* order = reinterpret_cast<uint32_t*>(sc);
    uint16_t* keys = reinterpret_cast<uint16_t*>(sc + ((tr.n_traces * 4 + 255) & ~(size_t)255));
    uint32_t* hist = reinterpret_cast<uint32_t*>(sc + ((tr.n_traces * 4 + 255) & ~(size_t)255) +
                                                 ((tr.n_traces * 2 + 255) & ~(size_t)255));
    cudaError_t e = cudaMemsetAsync(hist, 0, (kOrderKeys + 1) * 4, s);
    if (e != cudaSuccess) return e;
    const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((uint64_t)sm_count * 4,
                                                                             (tr.n_traces + 255) / 256));
    k_order_keys<<<grid, 256, 0, s>>>(P, keys, hist);
    k_order_scan<<<1, 1024, 0, s>>>(hist, tr.n_traces, force);
    k_order_scatter<<<grid, 256, 0, s>>>(keys, hist, order, tr.n_traces);
    return cudaGetLastError();
}

}  // namespace mig
