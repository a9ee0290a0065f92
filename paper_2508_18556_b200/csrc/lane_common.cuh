// lane_common.cuh — what the one-lane-per-(trace, policy) simulation kernels share (simulate_lane.cu,
// simulate_ff.cu, simulate_sa.cu): the launch parameters, the unit counters' layout, the decision-record hash step,
// the per-CTA totals reduction, and the grid size.
#pragma once

#include "device_common.cuh"

namespace mig {

struct LaneParams {
    const uint4* jobs;
    const uint4* ext;
    const uint64_t* off;
    const mig_job_estimate* est;
    uint64_t n_traces;
    mig_trace_result* out;
    mig_policy_totals* totals;
    unsigned long long* counter;
    const unsigned long long* est_err;  // error word of k_estimate (merged into this policy's totals)
    uint16_t* ring;                     // requeue FIFOs (job | need << 10) / Scheme A group lists, per lane
    const uint16_t* sid;                // mig_geometry::sid16: slot-level state id by occ | SM << 8 (FUSION_FISSION)
    const uint2* a7;                    // mig_geometry::a7, [state][n_a7] (FUSION_FISSION)
    uint4* pc;                          // PCIe contention: per lane and start slot, 2 x uint4 of run state (R39)
    unsigned long long* part;           // per-lane partial 64-bit totals, [CTA][kT64][kLaneThreads] (global scratch)
    const uint32_t* arr;                // arrival ticks aligned with jobs (R40), or NULL (batch)
    uint32_t n_a7;
    uint32_t ring_cap, max_jobs, ctx, n_pol_all, pol_idx;
    mig_policy pol;
    // k_ff_lane: tight fit against the ascending level memories (padded with 0xFFFFFFFF) read as constant-bank
    // operands, and the first profile of each level as nibbles (0xF = none)
    uint32_t lm[kMaxLevels];
    uint32_t lfirst;
    // Scheme A, grouped by k_sa_group before the launch (or NULL: the lane kernel's own grouping pass): the trace's
    // job records in group order (record x replaced by the job index) and per trace {5 group lengths, REJECT count,
    // error bits} + the decision hash after the t = 0 REJECT records
    const uint4* sa_desc;
    const uint4* sa_dext;
    const uint4* sa_hdr;
    // the order in which units are visited (trace_order.cu): unit u is trace order[u]; NULL = trace u
    const uint32_t* order;
};

// The trace of unit u, or ~0 once the units are exhausted (u >= n_traces).
__device__ __forceinline__ unsigned long long lane_unit_trace(const LaneParams& P, unsigned long long u) {
    return u >= P.n_traces ? ~0ull : P.order ? (unsigned long long)__ldg(P.order + u) : u;
}

constexpr int kLaneThreads = 128;
// Resident CTAs per SM (launch bounds) and where the u64 accumulators live: the Scheme B kernels (STATIC, DYNAMIC,
// FUSION_FISSION) keep them in shared memory, BASELINE and Scheme A in registers; every kind runs 8 CTAs (64
// registers). The per-lane partial totals live in global scratch, so 8 CTAs x 19.8 KB of shared memory still leave
// the L1 the table and record loads need. Measured A/B, config 2 / config 5 k_simulate: 4.84 / 250.7
// ms at 7 CTAs (BASELINE 6) with the partials in shared memory; 5.25 / 299 at 8 with them there (28 KB of L1); 4.80 /
// 240.6 at 8 with the partials in global scratch; 4.70 / 238.1 with BASELINE at 8 too (at 10 / 12 it spills: 4.87 /
// 5.66 on config 2); Scheme A at 7 / 8: 238.6 / 238.0 on config 5.
template <int KIND>
__host__ __device__ constexpr bool lane_acc_smem() { return KIND != MIG_BASELINE && KIND != MIG_SCHEME_A; }
template <int KIND>
__host__ __device__ constexpr int lane_min_blocks() { return 8; }
constexpr uint32_t kNoNeed = 0xFFu, kUnk = 0xFEu, kNoJob = 0xFFFFu;
constexpr uint32_t kNoEnd = 0xFFFFFFFFu;

// mig_policy_totals fields accumulated per CTA: 32-bit counts (index -> totals field; shared atomics, at most
// 2^32 / MIG_MAX_JOBS_PER_TRACE units per CTA) and 64-bit sums (per-lane partials). completed,
// restarts and energy are linear in these (n - rejected - failed; ooms - failed + preempts; idle_w * makespan +
// w_per_slice * busy) and are derived once per CTA.
constexpr int kT32 = 12, kT64 = 6;
// The per-trace counters are packed two per u32 (K0..K3: placements | creates, destroys | waits, rejected | ooms,
// preempts | failed), so each must stay below 2^16. A job runs at most 1 + 2 * kMaxLevels times (every OOM restart
// moves to a strictly larger memory level, R14; an early restart moves to a slice holding the converged forecast,
// R25, where it cannot preempt again before an OOM moves it up), so placements <= jobs * (1 + 2 * kMaxLevels);
// creates <= placements, destroys <= creates (only created instances are destroyed), and every WAIT is followed by
// an event or an arrival before the head is evaluated again, so waits <= placements + jobs.
static_assert((uint64_t)MIG_MAX_JOBS_PER_TRACE * (2 + 2 * kMaxLevels) < 65536,
              "packed 16-bit per-trace counters could overflow");
static __constant__ const uint8_t kF32[kT32] = {0, 1, 3, 4, 5, 6, 8, 9, 10, 11, 13, 20};
static __constant__ const uint8_t kF64[kT64] = {12, 15, 16, 17, 18, 19};

// FNV-1a-64 step on the two 32-bit halves of h (same as simulate.cu).
__device__ __forceinline__ void lrec(uint32_t& hl, uint32_t& hh, uint32_t tick, uint32_t lo) {
    const uint32_t x = hl ^ lo, y = hh ^ tick;
    const uint64_t p = (uint64_t)x * 0x1b3u;
    hl = (uint32_t)p;
    hh = (uint32_t)(p >> 32) + y * 0x1b3u + (x << 8);
}

// a12 per finished unit (k_ff_lane, k_simulate_lane): the lane's counts go to the CTA's 32-bit counters (c32, the
// kF32 order) by one shared reduction each, and its 64-bit sums to the lane's own partial slots in global scratch by
// one global reduction each. Plain RED instructions: no warp aggregation (lanes finish their units at different
// iterations, often one or two at a time) and no load on the lane's path.
__device__ __forceinline__ void lane_unit_totals(const LaneParams& P, uint32_t* c32, uint32_t n, uint32_t rejected,
                                                 uint32_t failed, uint32_t ooms, uint32_t preempts,
                                                 uint32_t placements, uint32_t waits, uint32_t creates,
                                                 uint32_t destroys, uint32_t makespan, uint32_t err,
                                                 unsigned long long turn, unsigned long long busy,
                                                 unsigned long long hash, unsigned long long mem,
                                                 unsigned long long waste) {
    const uint32_t cb = (uint32_t)__cvta_generic_to_shared(c32);
    const uint32_t v[10] = {1u, n, rejected, failed, ooms, preempts, placements, waits, creates, destroys};
#pragma unroll
    for (int k = 0; k < 10; ++k) asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(cb + 4 * k), "r"(v[k]) : "memory");
    asm volatile("red.shared.max.u32 [%0], %1;" ::"r"(cb + 40), "r"(makespan) : "memory");
    asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(cb + 44), "r"(err) : "memory");
    unsigned long long* d = P.part + (size_t)blockIdx.x * kT64 * kLaneThreads + threadIdx.x;
    const unsigned long long w[kT64] = {makespan, turn, busy, hash, mem, waste};
#pragma unroll
    for (int k = 0; k < kT64; ++k)
        asm volatile("red.global.add.u64 [%0], %1;" ::"l"(d + k * kLaneThreads), "l"(w[k]) : "memory");
}

// a12, once per CTA at the end of a launch: the policy's totals from the CTA's 32-bit counts (shared atomics,
// c32[kT32]) and its lanes' 64-bit partial sums (global scratch, [CTA][kT64][lane]); one thread per field, one
// atomic per field and CTA; completed, restarts and energy derived from them. Every thread of the CTA calls it.
__device__ __forceinline__ void lane_flush_totals(const LaneParams& P, const uint32_t* c32) {
    const uint32_t tid = threadIdx.x;
    __syncthreads();
    if (!P.totals) return;
    unsigned long long* dst = reinterpret_cast<unsigned long long*>(P.totals + P.pol_idx);
    if (tid == 0 && blockIdx.x == 0 && P.est_err && *P.est_err) atomicOr(dst + 20, *P.est_err);
    __shared__ unsigned long long red[24];
    if (tid < kT32 + kT64) {  // one thread per field reduces the CTA's lanes
        unsigned long long v = 0;
        if (tid < kT32) {
            v = c32[tid];
        } else {
            const unsigned long long* row = P.part + ((size_t)blockIdx.x * kT64 + (tid - kT32)) * kLaneThreads;
            for (int k = 0; k < kLaneThreads; ++k) v += __ldcg(row + k);  // written by global reductions (L2)
        }
        red[tid < kT32 ? kF32[tid] : kF64[tid - kT32]] = v;
    }
    __syncthreads();
    if (tid < 21) {
        unsigned long long v;
        if (tid == 2) v = red[1] - red[3] - red[4];  // completed
        else if (tid == 7) v = red[5] - red[4] + red[6];  // restarts
        else if (tid == 14) v = (unsigned long long)P.pol.idle_w * red[12] + (unsigned long long)P.pol.w_per_slice * red[16];
        else v = red[tid];
        if (v) {
            if (tid == 13) atomicMax(dst + 13, v);
            else if (tid == 20) atomicOr(dst + 20, v);
            else atomicAdd(dst + tid, v);
        }
    }
}

// Grid: resident CTAs per SM x SMs (persistent; units are taken from the counter), capped by the unit count.
inline uint64_t lane_blocks(int per_sm, uint64_t n_traces, int sm_count) {
    uint64_t blocks = (uint64_t)per_sm * sm_count;
    const uint64_t want = (n_traces + kLaneThreads - 1) / kLaneThreads;
    if (want < blocks) blocks = want;
    return blocks < 1 ? 1 : blocks;
}

// Launchers of the specialised lane kernels (simulate_ff.cu, simulate_sa.cu); max_blocks caps the grid (the
// per-lane scratch is sized for it).
cudaError_t launch_ff_lane(const DevGeom* Gdev, const LaneParams& P, uint32_t ns, uint64_t max_blocks, int sm_count,
                           cudaStream_t stream);
cudaError_t launch_base_lane(const DevGeom* Gdev, const LaneParams& P, uint64_t max_blocks, int sm_count,
                             cudaStream_t stream);
size_t trace_order_scratch_bytes(uint64_t n_traces);
cudaError_t launch_trace_order(const mig_traces& tr, const DevGeom* Gh, uint32_t ctx, void* buf, bool force,
                               int sm_count, cudaStream_t s);
cudaError_t launch_sa_group(const DevGeom* Gdev, const LaneParams& P, uint4* desc, uint4* dext, uint4* hdr,
                            int sm_count, cudaStream_t stream);

}  // namespace mig
