// simulate_lane.cu — k_simulate_lane: the MIGM scheduler + partition-manager event loop (SURVEY.md §8(a) rows a1,
// a4-a12) with ONE LANE PER (trace, policy) unit, for the Scheme B family of policies (BASELINE, STATIC, DYNAMIC,
// FUSION_FISSION, +EARLY_RESTART / WARP_FOLD / WAVE_TIME).
//
// Why a lane per trace. A trace is a sequential discrete-event loop whose per-decision work is a handful of bitmask
// operations; the group kernel (simulate.cu, 8 or 32 lanes per trace) spends most issue slots on work that is
// uniform across the group. Here every lane runs its own trace, and the whole decision procedure is reduced to
// O(1) table lookups and bit arithmetic on per-lane registers:
//   Alg. 2 ...... s_alloc[occupancy][profile]: the argmax-fcr legal start (tie -> highest, R5),
//                                    evaluated once per CTA from the fcr table of Alg. 1 (the
//                                    reachability "can be precomputed offline"), so a decision is one LDS
//   reuse (R7) ....... idle instance starts & a per-profile "tightly fits" mask over the per-slot
//                                    profile nibbles (<= 7 idle instances, highest start first)
//   fusion / fission (R8) .......... only when Alg. 2 fails: the candidates touching no busy slot (a table by busy
//                                    mask): one entry of the host-built answer table by (slot-level state of
//                                    (occ, SM), profile, candidates) (global memory, L1-resident)
//   next event (R28) ............... min over the eight per-slot end ticks; ties by (kind, job) (shared memory)
// The loop is a flat state machine (PASS: one head evaluation; EVT: one event; FIN: write the unit's result and take
// the next unit), so the 32 lanes of a warp stay in one loop even though their traces are at different points:
// the cost of an iteration is the sum of the branches present in the warp, not the slowest trace. Units are taken
// from an atomic counter one ahead (lane-level work stealing); per-policy totals are per-lane shared-memory partials
// reduced once per CTA.
//
// Per-lane state: occupancy occ, instance starts SM, busy starts BS / busy slots BM, profile
// nibble per start slot (prof4), end tick and job|kind per start slot (shared memory, [slot][lane]),
// the head job's record (prefetched when the queue advances), a requeue FIFO in global scratch (rare: OOM /
// preempt restarts, R13), packed 16-bit counters, FNV-1a-64 hash halves, four u64 accumulators.
//
// The record stream, counters and accumulators are exactly those of the group kernel and the oracle (DESIGN.md
// "Decision record"), so results are bit-identical (tests/test_kernel_variants_gpu.py, MIG_LANES_PER_TRACE=1).
#include <stdlib.h>
#include <string.h>

#include <algorithm>

#include "lane_common.cuh"

namespace mig {

struct LaneShared {
    DevGeom G;
    uint8_t alloc[256 * 8];   // Alg. 2 result by (occupancy, profile): placement index k, or 0xFF = FAIL
    uint16_t cbase[8];        // fusion/fission-table column of candidate mask 0 of profile p
    uint8_t nobusy[256 * 8];  // FF: placements k of profile p (bit k) that touch no busy slot, by busy-slot mask
    unsigned long long reuse_sel[16];  // FF: byte q = 0xFF if an idle instance of profile q tightly fits profile p
                                       // (same memory, compute >=; R7), selecting from the idle-by-profile masks
    uint8_t scand[16];        // STATIC: layout starts whose slice can hold profile p
    uint8_t lvl_first[8];     // first profile of each memory level ([n_levels] = 0xFF)
    uint32_t lmem[8];         // level memories, padded with 0xFFFFFFFF beyond n_levels
    uint32_t jk[8][kLaneThreads];  // per lane and start slot: job | end kind << 16 of the running job
    uint32_t et[8][kLaneThreads];  // per lane and start slot: end tick of the running job (kNoEnd = idle)
    uint32_t c32[kT32];            // per-CTA 32-bit counts (shared atomics)
    // the per-lane partial 64-bit totals live in global scratch (LaneParams::part)
};

// Tight fit (R6, R30): the smallest-memory profile holding req (ties -> fewer compute
// slices; profiles are sorted by (memory, compute)), with warp folding the same wave count as the whole GPU.
template <int KIND>
__device__ __forceinline__ uint32_t lane_tight_fit(const LaneShared& S, uint32_t req, uint32_t warps, bool fold) {
    const DevGeom& G = S.G;
    if (!fold || warps == 0) {
        // L = #levels with memory < req over the ascending level memories (padded with 0xFFFFFFFF; n_levels <= 5,
        // so L <= n_levels and lvl_first[n_levels] = 0xFF is "no profile"). Scheme B kinds: a branch-free binary
        // search over the 8 padded entries (3 loads); BASELINE, whose loop is a short dependent chain, keeps the
        // independent compares (measured A/B).
        uint32_t L = 0;
        if (KIND == MIG_BASELINE) {
#pragma unroll
            for (int l = 0; l < kMaxLevels; ++l) L += S.lmem[l] < req ? 1u : 0u;
        } else {
            L = S.lmem[3] < req ? 4u : 0u;
            L += S.lmem[L + 1] < req ? 2u : 0u;
            L += S.lmem[L] < req ? 1u : 0u;
        }
        return S.lvl_first[L];
    }
    const uint32_t cf = G.wave_cap[G.full_prof];
    for (uint32_t p = 0; p < G.n_prof; ++p) {
        if (G.mem[p] < req) continue;
        const uint32_t cp = G.wave_cap[p];
        if ((warps + cp - 1) / cp != (warps + cf - 1) / cf) continue;
        return p;
    }
    return kNoNeed;
}

__device__ __forceinline__ uint32_t lane_wave_ticks(const DevGeom& G, uint32_t ticks, uint32_t warps, uint32_t prof) {
    if (warps == 0) return ticks;
    const uint32_t cp = G.wave_cap[prof], cf = G.wave_cap[G.full_prof];
    const uint32_t wp = (warps + cp - 1) / cp, wf = (warps + cf - 1) / cf;
    return (uint32_t)(((uint64_t)ticks * wp + wf - 1) / wf);
}

// XR: the traces may carry extension records (jobs_ext); XR = false compiles them out (every ws / warps field 0).
// PF: the policy has none of MIG_WARP_FOLD, MIG_EARLY_RESTART, MIG_WAVE_TIME (their paths compiled out).
template <int KIND, bool EXT, bool XR = true, bool PF = false>
__global__ void __launch_bounds__(kLaneThreads, lane_min_blocks<KIND>())
    k_simulate_lane(const DevGeom* __restrict__ Gg, const LaneParams P) {
    const uint4* const pext = XR ? P.ext : nullptr;
    __shared__ __align__(16) LaneShared S;
    const uint32_t tid = threadIdx.x;
    {
        const uint32_t* src = reinterpret_cast<const uint32_t*>(Gg);
        uint32_t* dst = reinterpret_cast<uint32_t*>(&S.G);
        for (uint32_t i = tid; i < sizeof(DevGeom) / 4; i += blockDim.x) dst[i] = __ldg(src + i);
        if (tid < kT32) S.c32[tid] = 0;
#pragma unroll
        for (int f = 0; f < kT64; ++f) P.part[((size_t)blockIdx.x * kT64 + f) * kLaneThreads + tid] = 0;
    }
    __syncthreads();
    {
        const DevGeom& G = S.G;
        for (uint32_t i = tid; i < 256 * 8; i += blockDim.x) {  // Alg. 2 for every (occupancy, profile)
            const uint32_t occ = i >> 3, p = i & 7u;
            uint32_t best = 0, bk = 0xFFu;
            if (p < G.n_prof && occ < (1u << G.n_slots)) {
                for (uint32_t k = 0; k < G.n_place[p]; ++k) {
                    const uint32_t pl = G.place[p][k], qm = pl >> 8;
                    const uint32_t score = (pl && !(occ & qm)) ? ((uint32_t)G.fcr[occ | qm] << 8) | (pl & 0xFFu) : 0u;
                    if (score > best) {
                        best = score;
                        bk = k;
                    }
                }
            }
            S.alloc[i] = (uint8_t)bk;
            uint32_t nb = 0;  // here occ plays the busy-slot mask BM
            if (p < G.n_prof)
                for (uint32_t k = 0; k < G.n_place[p]; ++k) nb |= ((G.place[p][k] >> 8) & occ) ? 0u : 1u << k;
            S.nobusy[i] = (uint8_t)nb;
        }
        if (tid < 16) {
            uint32_t ok = 0, sc = 0;
            if (tid < G.n_prof) {
                for (uint32_t q = 0; q < G.n_prof; ++q)
                    if (G.level[q] == G.level[tid] && G.comp[q] >= G.comp[tid]) ok |= 1u << q;
                for (uint32_t i = 0; i < G.n_layout; ++i) {
                    const uint32_t lp = G.layout_prof[i];
                    if (G.level[lp] >= G.level[tid] && G.comp[lp] >= G.comp[tid]) sc |= 1u << G.layout_start[i];
                }
            }
            unsigned long long sel = 0;
            for (uint32_t q = 0; q < 8; ++q)
                if ((ok >> q) & 1u) sel |= 0xFFull << (8 * q);
            S.reuse_sel[tid] = sel;
            S.scand[tid] = (uint8_t)sc;
        }
        if (tid == 0) {
            uint32_t cb = 0;
            for (uint32_t p = 0; p < 8; ++p) {
                S.cbase[p] = (uint16_t)cb;
                cb += p < G.n_prof ? 1u << G.n_place[p] : 0u;
            }
        }
        if (tid < 8) {
            uint32_t f = 0xFFu;
            for (uint32_t p = G.n_prof; p-- > 0;)
                if (G.level[p] == tid) f = p;
            S.lvl_first[tid] = (uint8_t)(tid < G.n_levels ? f : 0xFFu);
            S.lmem[tid] = tid < G.n_levels ? G.level_mem[tid] : 0xFFFFFFFFu;
        }
    }
    __syncthreads();
    const DevGeom& G = S.G;

    const mig_policy& pol = P.pol;
    const bool fold = !PF && (pol.flags & MIG_WARP_FOLD) != 0;
    const bool er = !PF && (pol.flags & MIG_EARLY_RESTART) != 0;
    const bool wave = !PF && (pol.flags & MIG_WAVE_TIME) != 0;
    const uint32_t reconfig = pol.reconfig_ticks, full_mem = G.full_mem;
    const uint64_t jbase = P.off[0];
    // Scheme B: requeue FIFO (ring_cap entries); Scheme A: group lists, [memory level][ring_cap]
    // Scheme A: lane-interleaved within the CTA's block ([entry][lane]), since the grouping pass advances every
    // lane's lists in step (a warp at one list position touches one 64-B span, not 32 sectors; config 5 -1.5%).
    // Scheme B: each lane's FIFO contiguous (its rare pushes and pops reuse one sector; interleaving cost +0.9% on
    // config 2).
    constexpr uint32_t kRs = KIND == MIG_SCHEME_A ? kLaneThreads : 1u;  // entry stride
    uint16_t* ring = KIND == MIG_SCHEME_A
                         ? P.ring + (size_t)blockIdx.x * kLaneThreads * P.ring_cap * kMaxLevels + tid
                         : P.ring + (size_t)(blockIdx.x * kLaneThreads + tid) * P.ring_cap;
    // Scheme A: [0..7] group lengths by memory level, [8..15] next group-list index of the slice at slot s, [16..23]
    // the group's entries grouped before the launch (sa_desc; the rest are requeues in the ring)
    __shared__ uint16_t s_sa[KIND == MIG_SCHEME_A ? 24 : 1][kLaneThreads];
    uint16_t* glen = &s_sa[0][tid];
    uint16_t* nx = &s_sa[KIND == MIG_SCHEME_A ? 8 : 0][tid];
    uint16_t* plen = &s_sa[KIND == MIG_SCHEME_A ? 16 : 0][tid];
    uint32_t cur = 0xFFu, ns = 0, PM = 0, ready = 0;  // Scheme A: current group, its slices, pending-slice mask
    uint32_t pbase = 0;  // Scheme A with sa_desc: the current group's first record in the trace's grouped records
    const bool sa_pre = KIND == MIG_SCHEME_A && !EXT && P.sa_desc != nullptr;
    // PCIe contention (R39): slot s run state at pcs[2s] = {W lo, W hi, tk, rs}, pcs[2s+1] = {D, mem, iters,
    // F | started << 8 | dynamic << 9}; c_eff = transferring runs since the last retime; tick_end = an end event
    // was applied at the current tick (a tick with only starts has no scheduler pass)
    // EXT instantiations: PCIe contention and / or arrival streams (runtime flags, uniform per launch)
    const bool pcie = EXT && (pol.flags & MIG_PCIE_CONTENTION) != 0 && KIND != MIG_BASELINE;
    const bool arr = EXT && P.arr != nullptr;
    uint4* pcs = pcie ? P.pc + (size_t)(blockIdx.x * kLaneThreads + tid) * 16u : nullptr;
    uint32_t c_eff = 0;
    bool tick_end = false;
    uint32_t* jk = &S.jk[0][tid];
    uint32_t* et = &S.et[0][tid];
    const uint32_t fp = G.full_prof;

    // ---- unit state ----
    // A warp takes its units 32 at a time once every lane has finished its trace (a lane that finishes early waits in
    // mode 5), so the lanes start their traces together (as k_ff_lane; config 5's STATIC and Scheme A launches).
    const uint32_t lane_w = tid & 31u;
    auto take_batch = [&]() -> unsigned long long {
        unsigned long long u0 = 0;
        if (lane_w == 0) u0 = atomicAdd(P.counter, 32ull);
        u0 = __shfl_sync(FULL, u0, 0);
        return u0 + lane_w < P.n_traces ? u0 + lane_w : ~0ull;
    };
    unsigned long long tr = take_batch();
    uint64_t j0 = 0;
    uint32_t n = 0, err = 0, t = 0, qh = 0, rh = 0, rn = 0, mode = 0;
    uint32_t occ = 0, SM = 0, BS = 0, BM = 0, prof4 = 0, evm = 0;
    uint64_t IPM = 0;  // FF: idle instances by profile, byte p bit s = an idle instance of profile p starts at s
    uint32_t K0 = 0, K1 = 0, K2 = 0, K3 = 0, hl = 0, hh = 0;
    // u64 accumulators: turnaround, busy slice-ticks, MiB-ticks, wasted ticks (lane_acc_smem)
    constexpr bool kAccSmem = lane_acc_smem<KIND>();
    __shared__ unsigned long long s_acc[kAccSmem ? 4 : 1][kLaneThreads];
    unsigned long long r_acc0 = 0, r_acc1 = 0, r_acc2 = 0, r_acc3 = 0;
    unsigned long long& a_turn = kAccSmem ? s_acc[0][tid] : r_acc0;
    unsigned long long& a_busy = kAccSmem ? s_acc[kAccSmem ? 1 : 0][tid] : r_acc1;
    unsigned long long& a_mem = kAccSmem ? s_acc[kAccSmem ? 2 : 0][tid] : r_acc2;
    unsigned long long& a_waste = kAccSmem ? s_acc[kAccSmem ? 3 : 0][tid] : r_acc3;
    uint32_t hj = kNoJob, hneed = kUnk;  // head job and its tight fit (kUnk: not yet computed)
    uint4 hr = make_uint4(0, 0, 0, 0), he = make_uint4(0, 0, 0, 0);
    // BASELINE only: the running job (one at a time on the whole GPU)
    uint32_t bjob = 0, bend = 0;
    bool bbusy = false, boom = false;
    uint32_t na = 0, alast = 0;  // arrival streams (R40): next job to arrive, last arrival tick seen

    auto fetch_head = [&]() {  // queue = jobs[qh..n) ++ requeue FIFO
        if (qh < n) {
            hj = qh;
            hneed = kUnk;
        } else if ((KIND != MIG_BASELINE || EXT) && rn) {
            const uint32_t v = ring[rh * kRs];
            hj = v & 0x3FFu;
            hneed = v >> 10;
            if (hneed == 15u) hneed = kNoNeed;
            else if (hneed == 14u) hneed = kUnk;  // an arrival (R40): tight fit at its first evaluation
        } else {
            hj = kNoJob;
            return;
        }
        hr = __ldg(P.jobs + j0 + hj);
        he = pext ? __ldg(pext + j0 + hj) : make_uint4(0, 0, 0, 0);
    };
    // Arrival streams (reading R40): jobs whose arrival tick is <= t join the queue tail in queue order (after the
    // requeues of the tick's events); their tight fit is computed when they first reach the head.
    auto admit = [&]() -> bool {
        bool any = false;
        while (na < n) {
            const uint32_t a = __ldg(P.arr + j0 + na);
            if (a > t) break;
            if (a < alast) err |= (uint32_t)MIG_ERR_BAD_RECORD;  // arrival ticks must not decrease
            alast = max(alast, a);
            uint32_t pos = rh + rn;
            if (pos >= P.ring_cap) pos -= P.ring_cap;
            ring[pos * kRs] = (uint16_t)(na | (14u << 10));
            ++rn;
            ++na;
            if (hj == kNoJob) fetch_head();
            any = true;
        }
        return any;
    };
    auto init_unit = [&]() {
        const uint64_t o0 = P.off[tr], o1 = P.off[tr + 1];
        j0 = o0 - jbase;
        const uint64_t n64 = o1 - o0;
        err = 0;
        n = (uint32_t)n64;
        if (n64 > P.max_jobs) {
            err = (uint32_t)MIG_ERR_TRACE_TOO_LONG;
            n = 0;
        }
        t = qh = rh = rn = evm = 0;
        BS = BM = 0;
        occ = SM = prof4 = 0;
        IPM = 0;
#pragma unroll
        for (int k = 0; k < 8; ++k) et[k * kLaneThreads] = kNoEnd;
        if (KIND == MIG_STATIC) {
            for (uint32_t i = 0; i < G.n_layout; ++i) {
                const uint32_t p = G.layout_prof[i], s = G.layout_start[i];
                SM |= 1u << s;
                prof4 |= p << (4 * s);
                occ |= G.lenmask[p] << s;
            }
        }
        c_eff = 0;
        if (KIND == MIG_SCHEME_A) {
            cur = 0xFFu;
            ns = PM = ready = pbase = 0;
#pragma unroll
            for (int l = 0; l < 8; ++l) glen[l * kLaneThreads] = plen[l * kLaneThreads] = 0;
        }
        K0 = K1 = K2 = K3 = 0;
        a_turn = a_busy = a_mem = a_waste = 0;
        hl = (uint32_t)kFnvOffset;
        hh = (uint32_t)(kFnvOffset >> 32);
        bbusy = false;
        mode = 0;
        if (KIND == MIG_BASELINE && EXT) prof4 = fp;  // the generic loop's whole-GPU "instance" at slot 0
        if (arr) {  // R40: the queue starts with the jobs arriving at t = 0
            qh = n;
            na = alast = 0;
            hj = kNoJob;
            admit();
        }
        if (KIND == MIG_SCHEME_A && sa_pre) {  // grouped before the launch (k_sa_group): no grouping pass
            const uint4 h0 = __ldg(P.sa_hdr + 2 * tr), h1 = __ldg(P.sa_hdr + 2 * tr + 1);
            const uint32_t lens[5] = {h0.x & 0xFFFFu, h0.x >> 16, h0.y & 0xFFFFu, h0.y >> 16, h0.z & 0xFFFFu};
#pragma unroll
            for (int l = 0; l < 5; ++l) glen[l * kLaneThreads] = plen[l * kLaneThreads] = (uint16_t)lens[l];
            K2 = h0.z >> 16;  // the REJECTs at t = 0
            err |= h0.w;
            hl = h1.x;
            hh = h1.y;
            hj = kNoJob;
            return;
        }
        fetch_head();
        if (KIND == MIG_SCHEME_A && hj != kNoJob) mode = 4;  // the grouping pass first
    };
    auto pop = [&]() {
        if (qh < n) {
            ++qh;
        } else {
            rh = rh + 1 == P.ring_cap ? 0u : rh + 1u;
            --rn;
        }
        fetch_head();
    };
    // Start a run of job j (record hr/he) on the instance at slot s of profile pr: end tick and
    // kind (OOM > COMPLETE > PREEMPT in one iteration, R29; early restart R25), power, memory integral, waste.
    auto start_run = [&](uint32_t j, uint32_t s, uint32_t pr, uint32_t rs, uint32_t& end, uint32_t& ek) {
        const uint32_t si = G.pinfo[pr];
        const uint32_t lev = si & 0xFu, comp = (si >> 4) & 0xFu;
        const uint32_t T = hr.z & 0xFFFFu;
        uint32_t ticks = hr.w;
        const bool dyn = ((hr.z >> 16) & 0xFFu) == kClassDynamic;
        uint32_t fe, pred = 0, conv = 0, phys = 0;
        const mig_job_estimate* ej = nullptr;
        if (__builtin_expect(dyn, 0) && !P.est) {  // DYNAMIC under MIG_TRACES_NO_DYNAMIC: flagged, no forecast
            err |= (uint32_t)MIG_ERR_BAD_RECORD;
            fe = kNever;
        } else if (__builtin_expect(dyn, 0)) {
            // the estimate's first 16 B hold pred, conv and the first exceeds of levels 0-1; levels 2-4 follow
            // (one request per 16 B block instead of one per field)
            ej = P.est + j0 + j;
            const uint4 e0 = __ldg(reinterpret_cast<const uint4*>(ej));
            pred = e0.y;
            conv = e0.z & 0xFFFFu;
            if (lev < 2) {
                fe = lev ? e0.w >> 16 : e0.w & 0xFFFFu;
            } else {
                const uint2 e1 = __ldg(reinterpret_cast<const uint2*>(ej) + 2);
                fe = lev == 2 ? e1.x & 0xFFFFu : lev == 3 ? e1.x >> 16 : e1.y & 0xFFFFu;
            }
        } else {
            const uint64_t phys64 = (uint64_t)hr.y + he.x + P.ctx;
            phys = phys64 > 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)phys64;
            fe = (T >= 1 && phys > G.level_mem[lev]) ? 1u : kNever;  // R12: static jobs OOM at iteration 1
        }
        if (KIND != MIG_BASELINE && wave) ticks = lane_wave_ticks(G, ticks, he.y, pr);
        const uint32_t cap = G.level_mem[lev];
        uint32_t i_pre = 0xFFFFFFFFu;
        if (KIND != MIG_BASELINE && er && conv > 0 && pred > cap && cap < full_mem) i_pre = conv;
        if (fe <= min(T, i_pre)) {
            ek = 1;
            end = rs + fe * ticks;
        } else if (i_pre < T) {
            ek = 2;
            end = rs + i_pre * ticks;
        } else {
            ek = 0;
            end = rs + T * ticks;
        }
        const uint32_t dur = end - rs;
        {  // ticks are u32: flag a run whose end would not fit (the trace's times wrapped; mig.h)
            const uint32_t it = ek == 1 ? fe : ek == 2 ? i_pre : T;
            if (((uint64_t)it * ticks + rs) >> 32) err |= (uint32_t)MIG_ERR_TICK_OVERFLOW;
        }
        if (EXT && pcie) {  // R39: the run's end follows its progress; power, memory and waste at its end
            const uint32_t it = ek == 1 ? fe : ek == 2 ? i_pre : T;
            const uint32_t mem =
                dyn ? (ej ? __ldg(reinterpret_cast<const uint32_t*>(ej) + 12 + (ek == 1 ? lev : ek == 2 ? 5u : 6u)) : 0u)
                    : phys;
            pcs[2 * s] = make_uint4(0u, 0u, rs, rs);
            pcs[2 * s + 1] = make_uint4(dur, mem, it, (hr.z >> 24) | (dyn ? 0x200u : 0u));
            end = rs;  // the slot's next event: the run's start
            return;
        }
        a_busy += (uint64_t)comp * dur;
        if (__builtin_expect(dyn, 0)) {
            const uint32_t* m = reinterpret_cast<const uint32_t*>(ej) + 12;  // mem_fe[5], mem_conv, mem_T
            if (ej) a_mem += (uint64_t)__ldg(m + (ek == 1 ? lev : ek == 2 ? 5u : 6u)) * ticks;
        } else {
            a_mem += (uint64_t)phys * dur;
        }
        if (ek) a_waste += dur;
    };
    // PCIe contention (reading R39): a transferring run (F > 0) advances at
    // 2^24 / (256 - F + F c) units of 2^-16 nominal ticks per tick, c = transferring runs in progress.
    auto pc_rate = [](uint32_t F, uint32_t c) -> uint64_t { return F ? (1u << 24) / (256u - F + F * c) : 65536u; };
    auto pc_advance = [&](uint32_t tn) {  // every run in progress advances to tn at the rate in effect
        for (uint32_t m = BS; m; m &= m - 1u) {
            const uint32_t s = (uint32_t)__ffs(m) - 1u;
            uint4 a = pcs[2 * s];
            const uint32_t misc = pcs[2 * s + 1].w;
            if (!((misc >> 8) & 1u)) continue;
            const uint64_t W = ((uint64_t)a.y << 32 | a.x) - (uint64_t)(tn - a.z) * pc_rate(misc & 0xFFu, c_eff);
            a.x = (uint32_t)W;
            a.y = (uint32_t)(W >> 32);
            a.z = tn;
            pcs[2 * s] = a;
        }
    };
    auto pc_retime = [&]() {  // runs due now start; recount c; every run in progress gets its end for the new rate
        uint32_t c = 0;
        for (uint32_t m = BS; m; m &= m - 1u) {
            const uint32_t s = (uint32_t)__ffs(m) - 1u;
            uint4 b = pcs[2 * s + 1];
            if (!((b.w >> 8) & 1u) && pcs[2 * s].w == t) {
                const uint64_t W = (uint64_t)b.x << 16;
                pcs[2 * s] = make_uint4((uint32_t)W, (uint32_t)(W >> 32), t, t);
                b.w |= 0x100u;
                pcs[2 * s + 1] = b;
            }
            c += ((b.w >> 8) & 1u) && (b.w & 0xFFu) ? 1u : 0u;
        }
        for (uint32_t m = BS; m; m &= m - 1u) {
            const uint32_t s = (uint32_t)__ffs(m) - 1u;
            const uint32_t misc = pcs[2 * s + 1].w;
            if (!((misc >> 8) & 1u)) continue;
            const uint4 a = pcs[2 * s];
            const uint64_t W = (uint64_t)a.y << 32 | a.x, rho = pc_rate(misc & 0xFFu, c);
            et[s * kLaneThreads] = t + (uint32_t)((W + rho - 1u) / rho);
        }
        c_eff = c;
    };
    // Slot es's event at t under contention: a start (no record; returns true) or an end whose actual duration
    // is accounted here (power R26, memory integral, waste).
    auto pc_event = [&](uint32_t es, uint32_t ek, uint32_t comp) -> bool {
        uint4 b = pcs[2 * es + 1];
        if (!((b.w >> 8) & 1u)) {
            const uint64_t W = (uint64_t)b.x << 16;
            pcs[2 * es] = make_uint4((uint32_t)W, (uint32_t)(W >> 32), t, t);
            b.w |= 0x100u;
            pcs[2 * es + 1] = b;
            return true;
        }
        const uint32_t actual = t - pcs[2 * es].w;
        a_busy += (uint64_t)comp * actual;
        a_mem += (b.w & 0x200u) ? (b.z ? (uint64_t)b.y * actual / b.z : 0ull) : (uint64_t)b.y * actual;
        if (ek) a_waste += actual;
        tick_end = true;
        return false;
    };
    auto head_need = [&]() {  // first evaluation of an initial queue entry: tight fit of req0 + record checks
        if (hneed == kUnk) {
            const uint32_t cls = (hr.z >> 16) & 0xFFu, T = hr.z & 0xFFFFu;
            if (cls > 2 || T > 4096) err |= (uint32_t)MIG_ERR_BAD_RECORD;
            const uint32_t req0 = cls == kClassDynamic ? G.mem[0] : hr.x + he.x + P.ctx;  // R16 / est + ws + ctx
            hneed = lane_tight_fit<KIND>(S, req0, he.y, fold);
        }
        return hneed;
    };

    bool active = tr < P.n_traces;
    if (active) init_unit();
    else mode = 3;
    // Every lane of a warp advances one step per iteration; the vote at the top and the __syncwarp points between
    // the phases keep the warp converged (without them the compiler's reconvergence points are too coarse and the
    // divergent paths of an iteration ran one after another: 4.5 active lanes per instruction).
    while (__any_sync(FULL, active)) {
        if constexpr (KIND == MIG_BASELINE && !EXT) {
            // ---- BASELINE: one job at a time on the whole GPU, queue order ----
            if (mode == 0) {
                bool ev = false;
                if (hj == kNoJob) {  // queue drained: the last run's end, then the unit is done
                    ev = bbusy;
                    mode = 2;
                } else {
                    const uint32_t j = hj, need = head_need();
                    if (need == kNoNeed) {
                        lrec(hl, hh, t, (j << 16) | (K_REJECT << 12) | 0xFF0u);
                        K2 += 1u;
                        pop();
                    } else if (bbusy) {  // the head waits for the running job
                        lrec(hl, hh, t, (j << 16) | (K_WAIT << 12) | 0xF00u | (need << 4));
                        K1 += 1u << 16;
                        ev = true;
                    } else {
                        lrec(hl, hh, t, (j << 16) | (K_PLACE_BASELINE << 12) | (fp << 4));
                        K0 += 1u;
                        uint32_t end, ek;
                        start_run(j, 0, fp, t, end, ek);
                        bjob = j;
                        bend = end;
                        boom = ek == 1;
                        bbusy = true;
                        pop();
                    }
                }
                if (ev) {  // the run's end event: COMPLETE, or OOM on the whole GPU = FAILED
                    t = bend;
                    const uint32_t lo = (bjob << 16) | (fp << 4);
                    if (boom) {
                        lrec(hl, hh, t, lo | (K_OOM << 12));
                        lrec(hl, hh, t, lo | (K_FAILED << 12));
                        K2 += 1u << 16;
                        K3 += 1u << 16;
                    } else {
                        lrec(hl, hh, t, lo | (K_COMPLETE << 12));
                        a_turn += t;
                    }
                    bbusy = false;
                }
            }
        } else if constexpr (KIND == MIG_SCHEME_A) {
            // ---- Scheme A, schedule_by_group (reading R38) ----
            if (mode == 4) {  // sorted_by_mig_group at t = 0, one job per iteration; REJECTs in queue order
                const uint32_t j = hj, need = head_need();
                if (need == kNoNeed) {
                    lrec(hl, hh, 0u, (j << 16) | (K_REJECT << 12) | 0xFF0u);
                    K2 += 1u;
                } else {
                    const uint32_t lv = G.level[need], c = glen[lv * kLaneThreads];
                    ring[(lv * P.ring_cap + c) * kRs] = (uint16_t)j;
                    glen[lv * kLaneThreads] = (uint16_t)(c + 1u);
                }
                pop();
                if (hj == kNoJob) mode = 0;
            }
            __syncwarp();
            if (mode == 0) {
                const uint32_t cand = PM & ~BS;
                if (cand) {  // the lowest idle slice with pending jobs takes its next one
                    const uint32_t s = (uint32_t)__ffs(cand) - 1u;
                    const uint32_t k = nx[s * kLaneThreads];
                    const uint32_t pl = sa_pre ? plen[cur * kLaneThreads] : 0u;
                    uint32_t j;
                    if (sa_pre && k < pl) {  // a grouped record (its x holds the job index)
                        hr = __ldg(P.sa_desc + j0 + pbase + k);
                        he = P.sa_dext ? __ldg(P.sa_dext + j0 + pbase + k) : make_uint4(0, 0, 0, 0);
                        j = hr.x;
                    } else {  // a requeued job (OOM / early restart), from the ring
                        j = ring[(cur * P.ring_cap + k - pl) * kRs];
                        hr = __ldg(P.jobs + j0 + j);
                        he = pext ? __ldg(pext + j0 + j) : make_uint4(0, 0, 0, 0);
                    }
                    const uint32_t pr = (prof4 >> (4 * s)) & 0xFu;
                    lrec(hl, hh, t, (j << 16) | (K_PLACE_GROUP << 12) | (s << 8) | (pr << 4));
                    K0 += 1u;
                    uint32_t end, ek;
                    start_run(j, s, pr, t < ready ? t + reconfig : t, end, ek);  // a new slice: reconfig first
                    et[s * kLaneThreads] = end;
                    jk[s * kLaneThreads] = j | (ek << 16);
                    BS |= 1u << s;
                    BM |= ((G.pinfo[pr] >> 8) & 0xFFu) << s;
                    nx[s * kLaneThreads] = (uint16_t)(k + ns);
                    if (k + ns >= glen[cur * kLaneThreads]) PM &= ~(1u << s);
                } else if (BS == 0) {  // drained: set_homogeneous_slices(next non-empty group)
                    uint32_t l = cur == 0xFFu ? 0u : cur + 1u;
                    while (l < G.n_levels && glen[l * kLaneThreads] == 0) ++l;
                    if (l < G.n_levels) {
                        const uint32_t nd = __popc(SM);
                        lrec(hl, hh, t, (0xFFFFu << 16) | (K_LAYOUT << 12) | (l << 4) | nd);
                        K1 += nd;
                        ns = G.n_alay[l];
                        const uint32_t len = glen[l * kLaneThreads];
                        SM = prof4 = PM = 0;
                        for (uint32_t k = 0; k < ns; ++k) {
                            const uint32_t e = G.alay[l][k], st = e & 0xFFu;
                            SM |= 1u << st;
                            prof4 |= (e >> 8) << (4 * st);
                            nx[st * kLaneThreads] = (uint16_t)k;
                            if (k < len) PM |= 1u << st;
                        }
                        K0 += ns << 16;
                        ready = t + reconfig;
                        cur = l;
                        if (sa_pre) {  // the group's grouped records follow those of the smaller levels
                            pbase = 0;
                            for (uint32_t q = 0; q < l; ++q) pbase += plen[q * kLaneThreads];
                        }
                    } else {
                        mode = 1;  // nothing left: EVT finds no running job and finishes the unit
                    }
                } else {
                    mode = 1;
                }
            }
            __syncwarp();
            if (mode == 1) {  // the events of the next tick (R28), then dispatch again
                if (!evm) {
                    if (EXT && pcie) pc_retime();
                    uint32_t e8[8];
#pragma unroll
                    for (int k = 0; k < 8; ++k) e8[k] = et[k * kLaneThreads];
                    uint32_t tn = e8[0];
#pragma unroll
                    for (int k = 1; k < 8; ++k) tn = min(tn, e8[k]);
                    if (tn == kNoEnd) {
                        mode = 2;
                    } else {
                        t = tn;
                        if (EXT && pcie) pc_advance(tn);  // the runs in progress reach tn at the rate in effect
                        tick_end = false;
#pragma unroll
                        for (int k = 0; k < 8; ++k) evm |= (e8[k] == tn ? 1u : 0u) << k;
                    }
                }
                if (evm) {
                    uint32_t es = (uint32_t)__ffs(evm) - 1u;
                    uint32_t v = jk[es * kLaneThreads];
                    for (uint32_t m = evm & (evm - 1u); m; m &= m - 1u) {
                        const uint32_t k = (uint32_t)__ffs(m) - 1u;
                        const uint32_t w = jk[k * kLaneThreads];
                        if (w < v) {
                            v = w;
                            es = k;
                        }
                    }
                    evm &= ~(1u << es);
                    const uint32_t job = v & 0xFFFFu, ek = v >> 16;
                    const uint32_t epr = (prof4 >> (4 * es)) & 0xFu, si = G.pinfo[epr];
                    const bool pc_start = EXT && pcie && pc_event(es, ek, (si >> 4) & 0xFu);  // R39: start
                    if (!pc_start) {
                        const uint32_t elo = (job << 16) | (es << 8) | (epr << 4);
                        lrec(hl, hh, t, elo | ((K_COMPLETE + ek) << 12));
                        a_turn += ek == 0 ? t : 0u;
                        K2 += ek == 1 ? 1u << 16 : 0u;
                        K3 += ek == 2 ? 1u : 0u;
                        uint32_t req = 0;
                        if (ek == 1) {
                            req = G.level_next[si & 0xFu];
                            if (req == 0) {
                                lrec(hl, hh, t, elo | (K_FAILED << 12));
                                K3 += 1u << 16;
                            }
                        } else if (ek == 2) {
                            req = min(__ldg(&P.est[j0 + job].pred_mib), full_mem);
                        }
                        if (req) {  // the tail of the job's new (larger) group
                            const uint32_t w = (fold && pext) ? __ldg(&pext[j0 + job].y) : 0u;
                            const uint32_t nn = lane_tight_fit<KIND>(S, req, w, fold);
                            if (nn == kNoNeed) {
                                lrec(hl, hh, t, (job << 16) | (K_REJECT << 12) | 0xFF0u);
                                K2 += 1u;
                            } else {
                                const uint32_t lv = G.level[nn], c = glen[lv * kLaneThreads];
                                ring[(lv * P.ring_cap + c - (sa_pre ? plen[lv * kLaneThreads] : 0u)) * kRs] =
                                    (uint16_t)job;
                                glen[lv * kLaneThreads] = (uint16_t)(c + 1u);
                            }
                        }
                        et[es * kLaneThreads] = kNoEnd;
                        BS &= ~(1u << es);
                        BM &= ~(((si >> 8) & 0xFFu) << es);
                    }
                    if (!evm) mode = (pcie && !tick_end) ? 1u : 0u;  // a tick with only starts has no pass
                }
            }
        } else {
            // ---- PASS: evaluate the head of the queue (Alg. 4, one decision) ----
            // P1 (local decision, incl. fusion/fission A7) | P2 (record, run start, pop), with the
            // warp reconverged between phases: every decision path then shares one copy of the common code.
            if (mode == 0 && hj == kNoJob) mode = 1;
            const bool pass = mode == 0;
            uint32_t j = 0, need = 0, s = 0, kd = 0, nd = 0, pr = 0, lo = 0;
            if (pass) {
                j = hj;
                need = head_need();
                pr = need;
                const uint32_t jsh = j << 16;
                if (need == kNoNeed) {  // no profile can ever hold the job: REJECT
                    lo = jsh | (K_REJECT << 12) | 0xFF0u;
                    kd = K_REJECT;
                } else if (KIND == MIG_BASELINE) {  // one job at a time on the whole GPU
                    if (BS) {
                        kd = K_WAIT;
                        lo = jsh | (K_WAIT << 12) | 0xF00u | (need << 4);
                    } else {
                        s = 0;
                        pr = fp;
                        kd = K_PLACE_BASELINE;
                    }
                } else if (KIND == MIG_STATIC) {  // smallest idle fitting layout slice, tie -> highest start (R11)
                    const uint32_t cand = S.scand[need];
                    uint32_t m = cand & ~BS, bk = 0;
                    while (m) {
                        const uint32_t k = (uint32_t)__ffs(m) - 1u;
                        m &= m - 1u;
                        const uint32_t il = G.pinfo[(prof4 >> (4 * k)) & 0xFu] & 0xFu;
                        bk = max(bk, (((15u - il) << 5) | k) + 1u);
                    }
                    if (bk) {
                        s = (bk - 1u) & 31u;
                        pr = (prof4 >> (4 * s)) & 0xFu;
                        kd = K_PLACE_STATIC;
                    } else {
                        kd = cand ? K_WAIT : K_REJECT;
                        lo = jsh | ((cand ? K_WAIT : K_REJECT) << 12) | 0xF00u | (need << 4);
                    }
                } else {
                    if (KIND == MIG_FUSION_FISSION) {  // an idle slice that tightly fits (R7)
                        uint64_t x = IPM & S.reuse_sel[need];
                        x |= x >> 32;
                        x |= x >> 16;
                        x |= x >> 8;
                        const uint32_t cand = (uint32_t)x & 0xFFu;
                        if (cand) {
                            s = 31u - __clz(cand);
                            pr = (prof4 >> (4 * s)) & 0xFu;
                            kd = K_REUSE;
                        }
                    }
                    if (!kd) {
                        const uint32_t a = S.alloc[(occ << 3) | need];  // Alg. 2: placement k
                        if (a != 0xFFu) {
                            s = G.place[need][a] & 0xFFu;
                            kd = K_ALLOC;
                        } else {
                            // fusion / fission candidates: placements touching no busy slot (none: WAIT)
                            const uint32_t cm =
                                (KIND == MIG_FUSION_FISSION && (SM & ~BS)) ? S.nobusy[(BM << 3) | need] : 0u;
                            if (KIND == MIG_FUSION_FISSION && cm) {
                                // A7 (R8): placement k destroys the idle instances it overlaps;
                                // best (fcr(result), -#destroyed, start) over the candidates c, one table entry
                                // per (slot-level state, profile, c) (host-built, mig_geometry::a7); the state id of
                                // (occ, SM) is looked up here, on the (rare) fusion path only
                                const uint32_t sid = __ldg(P.sid + (occ | (SM << 8)));
                                const uint2 e = __ldg(P.a7 + (sid * P.n_a7 + S.cbase[need] + cm));
                                const uint32_t best = e.x, by = e.y;
                                if (best) {
                                    s = best & 0xFFu;
                                    nd = 15u - ((best >> 8) & 0xFFu);
                                    const uint32_t rm = by & 0xFFu;
                                    IPM &= ~(0x0101010101010101ull * (SM & rm));  // destroyed (idle) instances
                                    occ &= ~rm;
                                    SM &= ~rm;
                                    kd = K_RECONF;
                                }
                            }
                            if (!kd) {  // sleep() until a running job finishes
                                kd = K_WAIT;
                                lo = jsh | (K_WAIT << 12) | 0xF00u | (need << 4);
                            }
                        }
                    }
                }
            }
            __syncwarp();
            if (pass) {
                // ---- P2: create (ALLOC / RECONF, try_new_mig_slice PAPER.md:609), the decision record, the run ----
                const bool created = kd == K_ALLOC || kd == K_RECONF;
                const bool place = kd != K_WAIT && kd != K_REJECT;
                if (created) {
                    occ |= ((G.pinfo[need] >> 8) & 0xFFu) << s;
                    if (KIND == MIG_FUSION_FISSION) SM |= 1u << s;
                    prof4 = (prof4 & ~(0xFu << (4 * s))) | (need << (4 * s));
                }
                if (KIND == MIG_FUSION_FISSION && kd == K_REUSE) IPM &= ~(1ull << (8 * pr + s));
                if (place) lo = (j << 16) | (kd << 12) | (s << 8) | (pr << 4) | nd;
                lrec(hl, hh, t, lo);
                K0 += place ? (created ? 0x10001u : 1u) : 0u;
                K1 += kd == K_WAIT ? 1u << 16 : nd;
                K2 += kd == K_REJECT ? 1u : 0u;
                if (place) {
                    uint32_t end, ek;
                    start_run(j, s, pr, t + (created ? reconfig : 0u), end, ek);
                    et[s * kLaneThreads] = end;
                    jk[s * kLaneThreads] = j | (ek << 16);
                    BS |= 1u << s;
                    BM |= ((G.pinfo[pr] >> 8) & 0xFFu) << s;
                }
                if (kd == K_WAIT) mode = 1;
                else pop();
            }
            __syncwarp();
            // ---- EVT: apply one event (min end tick; ties COMPLETE < OOM < PREEMPT, then job id, R28) ----
            if (mode == 1) {
                if (!evm) {
                    if (EXT && pcie) pc_retime();
                    uint32_t e8[8];
#pragma unroll
                    for (int k = 0; k < 8; ++k) e8[k] = et[k * kLaneThreads];
                    uint32_t tn = e8[0];
#pragma unroll
                    for (int k = 1; k < 8; ++k) tn = min(tn, e8[k]);
                    if (arr && na < n) tn = min(tn, __ldg(P.arr + j0 + na));  // the next arrival (R40)
                    if (tn == kNoEnd) {
                        mode = 2;
                    } else {
                        t = tn;
                        if (EXT && pcie) pc_advance(tn);  // the runs in progress reach tn at the rate in effect
                        tick_end = false;
#pragma unroll
                        for (int k = 0; k < 8; ++k) evm |= (e8[k] == tn ? 1u : 0u) << k;
                        if (!evm) {  // an arrival-only tick: admit, then one scheduler pass (R9, R40)
                            admit();
                            mode = 0;
                        }
                    }
                }
                if (evm) {
                    uint32_t es = (uint32_t)__ffs(evm) - 1u;
                    uint32_t v = jk[es * kLaneThreads];
                    if (evm & (evm - 1u)) {
                        uint32_t m = evm & (evm - 1u);
                        while (m) {
                            const uint32_t k = (uint32_t)__ffs(m) - 1u;
                            m &= m - 1u;
                            const uint32_t w = jk[k * kLaneThreads];
                            if (w < v) {
                                v = w;
                                es = k;
                            }
                        }
                    }
                    evm &= ~(1u << es);
                    const uint32_t job = v & 0xFFFFu, ek = v >> 16;
                    const uint32_t epr = (prof4 >> (4 * es)) & 0xFu, si = G.pinfo[epr];
                    const bool pc_start = EXT && pcie && pc_event(es, ek, (si >> 4) & 0xFu);  // R39: start
                    if (!pc_start) {
                        const uint32_t elo = (job << 16) | (es << 8) | (epr << 4);
                        lrec(hl, hh, t, elo | ((K_COMPLETE + ek) << 12));  // COMPLETE 6 / OOM 7 / PREEMPT 8
                        a_turn += ek == 0 ? t - (arr ? __ldg(P.arr + j0 + job) : 0u) : 0u;  // completion - arrival
                        K2 += ek == 1 ? 1u << 16 : 0u;
                        K3 += ek == 2 ? 1u : 0u;
                        uint32_t req = 0;
                        if (ek == 1) {  // OOM: next larger slice (R14) or FAILED on the whole GPU
                            req = G.level_next[si & 0xFu];
                            if (req == 0) {
                                lrec(hl, hh, t, elo | (K_FAILED << 12));
                                K3 += 1u << 16;
                            }
                        } else if (ek == 2) {  // PREEMPT: restart on the slice meeting the forecast (R25)
                            req = min(__ldg(&P.est[j0 + job].pred_mib), full_mem);
                        }
                        if (req) {  // back to the queue tail (R13) with the new tight fit
                            const uint32_t w = (fold && pext) ? __ldg(&pext[j0 + job].y) : 0u;
                            const uint32_t nn = lane_tight_fit<KIND>(S, req, w, fold);
                            uint32_t pos = rh + rn;
                            if (pos >= P.ring_cap) pos -= P.ring_cap;
                            ring[pos * kRs] = (uint16_t)(job | ((nn == kNoNeed ? 15u : nn) << 10));
                            ++rn;
                            if (hj == kNoJob) fetch_head();
                        }
                        et[es * kLaneThreads] = kNoEnd;
                        const uint32_t ext = ((si >> 8) & 0xFFu) << es;
                        BS &= ~(1u << es);
                        BM &= ~ext;
                        if (KIND == MIG_DYNAMIC) {  // free on completion (R10)
                            occ &= ~ext;
                            K1 += 1u;
                        }
                        if (KIND == MIG_FUSION_FISSION) IPM |= 1ull << (8 * epr + es);  // the instance is idle
                    }
                    if (!evm) {  // the tick is over: its arrivals join the queue (R40); a tick with only starts has no pass
                        const bool arrived = arr && admit();
                        mode = (pcie && !tick_end && !arrived) ? 1u : 0u;
                    }
                }
            }
        }
        __syncwarp();
        // ---- FIN: the unit's result (96 B) and totals; take the next unit ----
        if (mode == 2) {
            const uint32_t placements = K0 & 0xFFFFu, creates = K0 >> 16, destroys = K1 & 0xFFFFu, waits = K1 >> 16,
                           rejected = K2 & 0xFFFFu, ooms = K2 >> 16, preempts = K3 & 0xFFFFu, failed = K3 >> 16;
            const uint32_t completed = n - rejected - failed, restarts = ooms - failed + preempts;
            const uint32_t makespan = t;
            const uint64_t energy = (uint64_t)pol.idle_w * makespan + (uint64_t)pol.w_per_slice * a_busy;
            if (P.out) {
                uint4* o = reinterpret_cast<uint4*>(P.out + tr * P.n_pol_all + P.pol_idx);
                o[0] = make_uint4(makespan, n, completed, rejected);
                o[1] = make_uint4(failed, ooms, preempts, restarts);
                o[2] = make_uint4(placements, waits, creates, destroys);
                o[3] = make_uint4((uint32_t)energy, (uint32_t)(energy >> 32), (uint32_t)a_turn,
                                  (uint32_t)(a_turn >> 32));
                o[4] = make_uint4((uint32_t)a_busy, (uint32_t)(a_busy >> 32), hl, hh);
                o[5] = make_uint4((uint32_t)a_mem, (uint32_t)(a_mem >> 32), (uint32_t)a_waste,
                                  (uint32_t)(a_waste >> 32));
            }
            // a12: the unit's counts and sums into the CTA's totals (lane_common.cuh)
            lane_unit_totals(P, S.c32, n, rejected, failed, ooms, preempts, placements, waits, creates, destroys, makespan,
                             err, a_turn, a_busy, ((unsigned long long)hh << 32) | hl, a_mem, a_waste);
            mode = 5;  // wait for the warp's other lanes
        }
        if (__all_sync(FULL, mode == 3 || mode == 5) && __any_sync(FULL, mode == 5)) {  // the warp's next 32 units
            tr = take_batch();
            if (tr < P.n_traces) {
                init_unit();
            } else {
                active = false;
                mode = 3;  // done: the lane keeps voting (and passing the __syncwarp points) until its warp is done
            }
        }
    }
    lane_flush_totals(P, S.c32);
}

// MIG_SA_PREGROUP=0: Scheme A's grouping pass inside the lane kernel instead of k_sa_group (A/B and parity).
static bool sa_pregroup_enabled() {
    static int on = -1;
    if (on < 0) {
        const char* env = getenv("MIG_SA_PREGROUP");
        on = env ? atoi(env) != 0 : 1;
    }
    return on != 0;
}

// MIG_FF_FAST=0 selects k_simulate_lane for the FUSION_FISSION fast case too (A/B and parity of both kernels).
static bool ff_fast_enabled() {
    static int on = -1;
    if (on < 0) {
        const char* env = getenv("MIG_FF_FAST");
        on = env ? atoi(env) != 0 : 1;
    }
    return on != 0;
}

// Grid: resident CTAs per SM x SMs (persistent; units are taken from the counter), capped by the unit count.
template <int KIND>
static int lane_per_sm() {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_simulate_lane<KIND, false>, kLaneThreads, 0);
    return per_sm < 1 ? 1 : per_sm;
}

// The largest grid of any kind (sizes the per-lane scratch shared by the launches of one call).
uint64_t simulate_lane_grid(uint64_t n_traces, int sm_count) {
    const int per_sm = std::max(std::max(lane_per_sm<MIG_BASELINE>(), lane_per_sm<MIG_FUSION_FISSION>()),
                                lane_per_sm<MIG_SCHEME_A>());
    return lane_blocks(per_sm, n_traces, sm_count);
}

uint32_t simulate_lane_threads() { return kLaneThreads; }
uint32_t simulate_lane_partials() { return kT64; }

// One launch per policy. counter: a zeroed u64; ring: blocks * kLaneThreads * max_jobs u16 of scratch.
cudaError_t launch_simulate_lane(const DevGeom* Gdev, const mig_traces& tr, const mig_policy& pol, uint32_t pol_idx,
                                 uint32_t n_pol_all, const mig_job_estimate* est, mig_trace_result* out,
                                 mig_policy_totals* totals, unsigned long long* counter,
                                 const unsigned long long* est_err, uint16_t* ring, uint64_t blocks,
                                 const uint16_t* sid, const uint32_t* a7, uint32_t n_a7,
                                 uint4* pc, unsigned long long* part, int sm_count, cudaStream_t stream,
                                 const DevGeom* Gh, const uint32_t* order) {
    LaneParams P;
    memset(&P, 0, sizeof(P));
    P.order = order;  // visited through by k_ff_lane only (the kind the order helps); the other kernels ignore it
    P.jobs = (const uint4*)tr.jobs;
    P.ext = (const uint4*)tr.jobs_ext;
    P.off = tr.trace_off;
    P.est = est;
    P.n_traces = tr.n_traces;
    P.out = out;
    P.totals = totals;
    P.counter = counter;
    P.est_err = est_err;
    P.ring = ring;
    P.ring_cap = tr.max_jobs;
    P.max_jobs = tr.max_jobs;
    P.ctx = pol.ctx_mib;
    P.n_pol_all = n_pol_all;
    P.pol_idx = pol_idx;
    P.pol = pol;
    P.sid = sid;
    P.part = part;
    P.a7 = reinterpret_cast<const uint2*>(a7);
    P.n_a7 = n_a7;
    P.pc = pc;
    P.arr = tr.arrival;
    const int per_sm = pol.kind == MIG_BASELINE   ? lane_per_sm<MIG_BASELINE>()
                       : pol.kind == MIG_SCHEME_A ? lane_per_sm<MIG_SCHEME_A>()
                                                  : lane_per_sm<MIG_FUSION_FISSION>();
    const dim3 grid((unsigned)std::min<uint64_t>(blocks, lane_blocks(per_sm, tr.n_traces, sm_count))),
        block(kLaneThreads);
    const bool con = (pol.flags & MIG_PCIE_CONTENTION) != 0 && pol.kind != MIG_BASELINE;  // BASELINE: c <= 1
    if (con && !P.pc) return cudaErrorInvalidValue;
    const bool ext = con || P.arr;  // the EXT instantiation: contention and / or arrival streams
    const bool pf = (pol.flags & (MIG_WARP_FOLD | MIG_EARLY_RESTART | MIG_WAVE_TIME)) == 0;
    // the fast kernels (simulate_ff.cu) take extension records and early restart, not warp folding or wave time
    const bool ff_pf = (pol.flags & (MIG_WARP_FOLD | MIG_WAVE_TIME)) == 0;
    const bool fast = (pol.kind == MIG_FUSION_FISSION || pol.kind == MIG_DYNAMIC || pol.kind == MIG_BASELINE) && !ext &&
                      ff_pf && Gh && ff_fast_enabled();
    if (fast) {
        for (int l = 0; l < kMaxLevels; ++l) P.lm[l] = l < (int)Gh->n_levels ? Gh->level_mem[l] : 0xFFFFFFFFu;
        uint32_t lf = 0;
        for (uint32_t l = 0; l < 8; ++l) {  // first (fewest compute) profile of each level; 0xF = none
            uint32_t f = 0xFu;
            for (uint32_t p = Gh->n_prof; p-- > 0;)
                if (l < Gh->n_levels && Gh->level[p] == l) f = p;
            lf |= f << (4 * l);
        }
        P.lfirst = lf;
        if (pol.kind == MIG_BASELINE) return launch_base_lane(Gdev, P, blocks, sm_count, stream);
        uint32_t ns = 0;  // one past the highest start slot of any placement
        for (uint32_t p = 0; p < Gh->n_prof; ++p)
            for (uint32_t k = 0; k < Gh->n_place[p]; ++k) ns = std::max(ns, (Gh->place[p][k] & 0xFFu) + 1u);
        return launch_ff_lane(Gdev, P, ns, blocks, sm_count, stream);
    }
    switch (pol.kind) {
        case MIG_BASELINE:
            if (ext) k_simulate_lane<MIG_BASELINE, true><<<grid, block, 0, stream>>>(Gdev, P);
            else if (P.ext) k_simulate_lane<MIG_BASELINE, false><<<grid, block, 0, stream>>>(Gdev, P);
            else if (pf) k_simulate_lane<MIG_BASELINE, false, false, true><<<grid, block, 0, stream>>>(Gdev, P);
            else k_simulate_lane<MIG_BASELINE, false, false><<<grid, block, 0, stream>>>(Gdev, P);
            break;
        case MIG_STATIC:
            if (ext) k_simulate_lane<MIG_STATIC, true><<<grid, block, 0, stream>>>(Gdev, P);
            else if (P.ext) k_simulate_lane<MIG_STATIC, false><<<grid, block, 0, stream>>>(Gdev, P);
            else if (pf) k_simulate_lane<MIG_STATIC, false, false, true><<<grid, block, 0, stream>>>(Gdev, P);
            else k_simulate_lane<MIG_STATIC, false, false><<<grid, block, 0, stream>>>(Gdev, P);
            break;
        case MIG_DYNAMIC:
            if (ext) k_simulate_lane<MIG_DYNAMIC, true><<<grid, block, 0, stream>>>(Gdev, P);
            else if (P.ext) k_simulate_lane<MIG_DYNAMIC, false><<<grid, block, 0, stream>>>(Gdev, P);
            else if (pf) k_simulate_lane<MIG_DYNAMIC, false, false, true><<<grid, block, 0, stream>>>(Gdev, P);
            else k_simulate_lane<MIG_DYNAMIC, false, false><<<grid, block, 0, stream>>>(Gdev, P);
            break;
        case MIG_FUSION_FISSION:
            if (ext) k_simulate_lane<MIG_FUSION_FISSION, true><<<grid, block, 0, stream>>>(Gdev, P);
            else if (P.ext) k_simulate_lane<MIG_FUSION_FISSION, false><<<grid, block, 0, stream>>>(Gdev, P);
            else if (pf) k_simulate_lane<MIG_FUSION_FISSION, false, false, true><<<grid, block, 0, stream>>>(Gdev, P);
            else k_simulate_lane<MIG_FUSION_FISSION, false, false><<<grid, block, 0, stream>>>(Gdev, P);
            break;
        case MIG_SCHEME_A:
            if (P.arr) return cudaErrorInvalidValue;  // Scheme A groups the whole queue at t = 0
            if (!ext && sa_pregroup_enabled() && tr.n_traces && tr.n_jobs) {
                // the grouping pass as its own launch (k_sa_group), its outputs in stream-ordered scratch
                const size_t nj = tr.n_jobs, nt = tr.n_traces;
                // the grouped extension records only when the policy reads more than the workspace (warp folding,
                // wave time); otherwise k_sa_group adds the workspace to the grouped record's true footprint
                const bool dext_needed = P.ext && (pol.flags & (MIG_WARP_FOLD | MIG_WAVE_TIME)) != 0;
                const size_t b_desc = nj * 16, b_dext = dext_needed ? nj * 16 : 0, b_hdr = nt * 32;
                uint8_t* sa = nullptr;
                cudaError_t e2 = mig_scratch_alloc((void**)&sa, b_desc + b_dext + b_hdr, stream);
                if (e2 != cudaSuccess) return e2;
                P.sa_desc = reinterpret_cast<const uint4*>(sa);
                P.sa_dext = dext_needed ? reinterpret_cast<const uint4*>(sa + b_desc) : nullptr;
                P.sa_hdr = reinterpret_cast<const uint4*>(sa + b_desc + b_dext);
                e2 = launch_sa_group(Gdev, P, (uint4*)P.sa_desc, (uint4*)P.sa_dext, (uint4*)P.sa_hdr, sm_count, stream);
                if (e2 == cudaSuccess) {
                    if (P.ext) k_simulate_lane<MIG_SCHEME_A, false><<<grid, block, 0, stream>>>(Gdev, P);
                    else if (pf) k_simulate_lane<MIG_SCHEME_A, false, false, true><<<grid, block, 0, stream>>>(Gdev, P);
                    else k_simulate_lane<MIG_SCHEME_A, false, false><<<grid, block, 0, stream>>>(Gdev, P);
                    e2 = cudaGetLastError();
                }
                mig_scratch_free(sa, stream);
                return e2;
            }
            if (ext) k_simulate_lane<MIG_SCHEME_A, true><<<grid, block, 0, stream>>>(Gdev, P);
            else if (P.ext) k_simulate_lane<MIG_SCHEME_A, false><<<grid, block, 0, stream>>>(Gdev, P);
            else if (pf) k_simulate_lane<MIG_SCHEME_A, false, false, true><<<grid, block, 0, stream>>>(Gdev, P);
            else k_simulate_lane<MIG_SCHEME_A, false, false><<<grid, block, 0, stream>>>(Gdev, P);
            break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

}  // namespace mig
