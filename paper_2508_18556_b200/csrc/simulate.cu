// simulate.cu — k_simulate: the MIGM scheduler + partition-manager event loop over many independent traces
// (SURVEY.md §8(a) rows a1, a4-a12).
//
// One warp per trace (persistent CTAs, atomic trace counter). The trace's jobs are staged into shared memory
// (coalesced 128-bit loads, 32 B per job: iterations, class, tight-fit profile, iteration ticks, first
// requirement, warps, forecast, convergence iteration and the first-exceed iteration of every memory level).
// The partition state is held in registers:
//   lane s (s < slots) ...... the instance that starts at memory slot s: packed profile info (memory level,
//                             compute, slot mask, profile id, valid/busy bits), end tick, job and end kind
//   warp-uniform ............ occupancy bitmask occ, instance-start mask SM, instance-end mask EM, busy-slot
//                             mask BM (fusion/fission and busy tests are bit arithmetic, no shuffles)
// Every decision is lane-parallel:
//   reuse / static choice ... __ballot_sync over instances (+ __clz for the highest start)
//   Alg. 2 lane k scores placement k as (fcr[occ|mask] << 8 | start) from the shared-memory
//                             fcr table; __reduce_max_sync picks the argmax, ties to the highest start (R5)
//   fusion / fission ........ lane k scores (fcr[occ'] << 16 | (15 - #destroyed) << 8 | start), occ' from the
//                             instance boundaries around placement k (R8)
//   next event .............. __reduce_min_sync over busy instances' end ticks; ties by (kind, job) (R28)
// The policy kind is a template parameter (no per-decision policy branches). Counters are packed 16-bit fields
// in four warp-uniform registers; the decision stream is folded into an FNV-1a-64 hash. Per-trace results
// (80 B) are written with 128-bit stores; per-policy totals are reduced in shared memory and added to global
// memory once per CTA.
#include <stdlib.h>
#include <string.h>

#include <mutex>

#include "device_common.cuh"

namespace mig {

struct SimParams {
    const uint4* jobs;
    const uint4* ext;
    const uint64_t* off;
    const mig_job_estimate* est;
    uint64_t n_traces;
    mig_trace_result* out;
    mig_policy_totals* totals;
    unsigned long long* counter;
    const unsigned long long* est_err;  // error word of k_estimate (merged into the totals)
    uint32_t max_jobs, n_pol, ctx;
    uint32_t ring_cap;  // = max_jobs
    uint32_t scheme_a;  // this launch runs the MIG_SCHEME_A policies (group lists are staged)
    uint32_t n_pol_all; // policies of the mig_simulate call (result stride)
    uint32_t pol_idx[kMaxPolicies];  // caller index of each policy of this launch
    mig_policy pol[kMaxPolicies];
};

constexpr size_t kGeomBytes = (sizeof(DevGeom) + 15) & ~size_t(15);
constexpr size_t kPolBytes = (kMaxPolicies * sizeof(mig_policy) + 15) & ~size_t(15);
constexpr int kTotFields = 24;  // mig_policy_totals
constexpr size_t kTotBytes = kMaxPolicies * kTotFields * 8;
constexpr uint32_t kValid = 1u << 31, kBusy = 1u << 30;

// A lane group of GW lanes simulates one trace (GW = 32: one trace per warp; GW = 8: four traces per warp).
// Group-scoped warp intrinsics: the member mask is the group's lanes, so groups of one warp may diverge.
template <int GW>
struct Grp {
    uint32_t gl, gbase, gmask;
    __device__ __forceinline__ explicit Grp(uint32_t lane) {
        gl = lane & (GW - 1);
        gbase = lane - gl;
        gmask = GW == 32 ? FULL : (((1u << (GW & 31)) - 1u) << gbase);
    }
    __device__ __forceinline__ uint32_t ballot(bool p) const { return __ballot_sync(gmask, p) >> gbase; }
    __device__ __forceinline__ uint32_t max(uint32_t v) const { return __reduce_max_sync(gmask, v); }
    __device__ __forceinline__ uint32_t min(uint32_t v) const { return __reduce_min_sync(gmask, v); }
    __device__ __forceinline__ uint32_t bor(uint32_t v) const { return __reduce_or_sync(gmask, v); }
    __device__ __forceinline__ uint32_t shfl(uint32_t v, uint32_t src) const { return __shfl_sync(gmask, v, src, GW); }
    __device__ __forceinline__ unsigned long long shfl64(unsigned long long v, uint32_t src) const {
        return __shfl_sync(gmask, v, src, GW);
    }
    __device__ __forceinline__ void sync() const { __syncwarp(gmask); }
};

// Same, one lane (staging: lanes over jobs).
__device__ __forceinline__ uint32_t tight_fit_lane(const DevGeom& G, uint32_t req, uint32_t warps, bool fold) {
    const uint32_t cf = G.wave_cap[G.full_prof];
    for (uint32_t p = 0; p < G.n_prof; ++p) {
        if (G.mem[p] < req) continue;
        if (fold && warps > 0) {
            uint32_t cp = G.wave_cap[p];
            if ((warps + cp - 1) / cp != (warps + cf - 1) / cf) continue;
        }
        return p;
    }
    return 0xFFu;
}

// Iteration time on profile p (flag MIG_WAVE_TIME, R31 variant): ticks are full-GPU times; a job of W warps runs
// waves(W, p) = ceil(W / wave_cap[p]) waves, so one iteration takes ceil(ticks * wp / wf) ticks.
__device__ __forceinline__ uint32_t wave_ticks(const DevGeom& G, uint32_t ticks, uint32_t warps, uint32_t prof) {
    if (warps == 0) return ticks;
    const uint32_t cp = G.wave_cap[prof], cf = G.wave_cap[G.full_prof];
    const uint32_t wp = (warps + cp - 1) / cp, wf = (warps + cf - 1) / cf;
    return (uint32_t)(((uint64_t)ticks * wp + wf - 1) / wf);
}

// Run accounting on the lane-distributed accumulators: busy slice-ticks, memory integral, wasted time.
__device__ __forceinline__ void acc_run(uint64_t& acc, uint32_t lane, uint64_t busy, uint64_t mem, uint64_t wasted) {
    acc += lane == 1 ? busy : lane == 2 ? mem : lane == 3 ? wasted : 0ull;
}

// FNV-1a-64 step h = (h ^ (tick << 32 | lo)) * (2^40 + 0x1b3) mod 2^64, on the two 32-bit halves of h.
__device__ __forceinline__ void rec(uint32_t& hl, uint32_t& hh, uint32_t tick, uint32_t lo) {
    const uint32_t x = hl ^ lo, y = hh ^ tick;
    const uint64_t p = (uint64_t)x * 0x1b3u;
    hl = (uint32_t)p;
    hh = (uint32_t)(p >> 32) + y * 0x1b3u + (x << 8);
}

// Occupied slots of the instances a placement [lo, hi] overlaps, expanded to their boundaries (FF only).
__device__ __forceinline__ uint32_t overlap_extent(uint32_t occ, uint32_t SM, uint32_t EM, uint32_t lo, uint32_t hi) {
    const uint32_t a = ((occ >> lo) & 1u) ? 31u - __clz(SM & ((2u << lo) - 1u)) : lo;
    const uint32_t b = ((occ >> hi) & 1u) ? (uint32_t)__ffs(EM & ~((1u << hi) - 1u)) - 1u : hi;
    return occ & ((2u << b) - 1u) & ~((1u << a) - 1u);
}

// Staged jobs of one trace in shared memory.
//   WIDE (32 B/job, short traces): A = {T | cls<<16 | need<<24, ticks, req0, warps},
//                                  B = {pred, conv | fe0<<16, fe1 | fe2<<16, fe3 | fe4<<16}
//   NARROW (16 B/job, long traces): A = {T | cls<<16 | need<<24, ticks, phys (STATIC/MODEL) | pred (DYNAMIC),
//                                  conv (DYNAMIC)}; the first-exceed iterations of a DYNAMIC job are read from
//                                  the estimate buffer at run start, req0 and warps from the trace records.
template <bool WIDE>
struct JobStore {
    uint4* A;
    const uint4* B;
    const uint4* gjobs;  // this trace's records (global)
    const uint4* gext;
    const mig_job_estimate* gest;
    uint32_t ctx;

    __device__ __forceinline__ uint32_t need(uint32_t j) const { return A[j].x >> 24; }
    __device__ __forceinline__ void set_need(uint32_t j, uint32_t nd) const {
        A[j].x = (A[j].x & 0x00FFFFFFu) | (nd << 24);
    }
    __device__ __forceinline__ uint32_t warps(uint32_t j) const {
        return WIDE ? A[j].w : (gext ? __ldg(&gext[j].y) : 0u);
    }
    __device__ __forceinline__ uint32_t pred(uint32_t j) const { return WIDE ? B[j].x : A[j].z; }
    // Memory integral of a run in MiB x ticks: a constant footprint times the run's duration, or
    // for a DYNAMIC job the estimator's prefix sum over the iterations it ran (ek: 0 COMPLETE after T,
    // 1 OOM after fe, 2 PREEMPT after conv) times the iteration ticks.
    __device__ __forceinline__ uint64_t run_mem(uint32_t j, uint32_t phys, uint32_t lev, uint32_t ek, uint32_t dur,
                                                uint32_t ticks) const {
        if (__builtin_expect(((A[j].x >> 16) & 0xFFu) != kClassDynamic, 1)) return (uint64_t)phys * dur;
        const uint32_t* m = reinterpret_cast<const uint32_t*>(gest + j) + 12;  // mem_fe[5], mem_conv, mem_T
        return (uint64_t)__ldg(m + (ek == 1 ? lev : ek == 2 ? 5u : 6u)) * ticks;
    }
    // NARROW only: requeue FIFO as a linked list through the spare high half of A[j].w
    __device__ __forceinline__ uint32_t next(uint32_t j) const { return A[j].w >> 16; }
    __device__ __forceinline__ void set_next(uint32_t j, uint32_t nx) const { A[j].w = (A[j].w & 0xFFFFu) | (nx << 16); }
    // T, ticks, first-exceed iteration of memory level lev, converged forecast (pred, conv; conv = 0 if none)
    // phys: the constant footprint of a STATIC/MODEL job (0 for DYNAMIC) for the memory integral.
    __device__ __forceinline__ void run_info(const DevGeom& G, uint32_t j, uint32_t lev, uint32_t& T, uint32_t& ticks,
                                             uint32_t& fe, uint32_t& pred, uint32_t& conv, uint32_t& phys) const {
        const uint4 a = A[j];
        T = a.x & 0xFFFFu;
        ticks = a.y;
        const bool dyn = ((a.x >> 16) & 0xFFu) == kClassDynamic;
        if (WIDE) {
            const uint4 b = B[j];
            pred = b.x;
            conv = b.y & 0xFFFFu;
            fe = reinterpret_cast<const uint16_t*>(&B[j])[3 + lev];
            phys = dyn ? 0u : b.x;
        } else {
            pred = 0;
            conv = 0;
            phys = a.z;
            fe = (T >= 1 && a.z > G.level_mem[lev]) ? 1u : kNever;  // R12: static jobs OOM at iteration 1
            if (__builtin_expect(dyn, 0)) {  // a real branch, not predicated
                pred = a.z;
                conv = a.w & 0xFFFFu;
                phys = 0;
                fe = __ldg(reinterpret_cast<const unsigned short*>(gest + j) + 6 + lev);
            }
        }
    }
};

struct TraceOut {
    uint32_t K0, K1, K2, K3;  // placements|creates<<16, destroys|waits<<16, rejected|ooms<<16, preempts|failed<<16
    uint64_t acc;             // lane-distributed: lane 0 turnaround, 1 busy slice-ticks, 2 MiB-ticks, 3 wasted ticks
    uint32_t hl, hh;          // decision hash halves
    uint32_t makespan;
};

// BASELINE: the non-partitioned GPU runs one job at a time in queue order, so there is no
// partition state and no requeue (an OOM on the whole GPU is FAILED). Straight-line code producing the same
// decision/event record stream as the general loop: [REJECT]* PLACE [REJECT]* WAIT <event> PLACE ...
template <bool WIDE>
__device__ __forceinline__ TraceOut baseline_trace(const DevGeom& G, uint32_t n, const JobStore<WIDE>& J,
                                                   uint32_t lane) {
    TraceOut o;
    o.K0 = o.K1 = o.K2 = o.K3 = 0;
    o.acc = 0;
    o.hl = (uint32_t)kFnvOffset;
    o.hh = (uint32_t)(kFnvOffset >> 32);
    const uint32_t fp = G.full_prof, pi = G.pinfo[fp];
    const uint32_t lev = pi & 0xFu, comp = (pi >> 4) & 0xFu;
    const uint32_t place_lo = (K_PLACE_BASELINE << 12) | (fp << 4);  // slot 0
    const uint32_t ev_lo = fp << 4;
    uint32_t t = 0, qh = 0;
    while (qh < n) {
        uint32_t j = qh, need = J.need(j);
        if (need == 0xFFu) {  // no profile can hold the job
            rec(o.hl, o.hh, t, (j << 16) | (K_REJECT << 12) | 0xFF0u);
            o.K2 += 1u;
            ++qh;
            continue;
        }
        rec(o.hl, o.hh, t, (j << 16) | place_lo);
        o.K0 += 1u;
        uint32_t T, ticks, fe, pred, conv, phys;
        J.run_info(G, j, lev, T, ticks, fe, pred, conv, phys);
        const bool oom = fe <= T;  // first exceed of the whole GPU (R12); no early restart on baseline
        const uint32_t end = t + (oom ? fe : T) * ticks;
        acc_run(o.acc, lane, (uint64_t)comp * (end - t), J.run_mem(j, phys, lev, oom ? 1u : 0u, end - t, ticks),
                oom ? end - t : 0u);
        ++qh;
        while (qh < n) {  // the rest of the pass at t: rejections, then the head waits
            const uint32_t need2 = J.need(qh);
            if (need2 == 0xFFu) {
                rec(o.hl, o.hh, t, (qh << 16) | (K_REJECT << 12) | 0xFF0u);
                o.K2 += 1u;
                ++qh;
                continue;
            }
            rec(o.hl, o.hh, t, (qh << 16) | (K_WAIT << 12) | 0xF00u | (need2 << 4));
            o.K1 += 1u << 16;
            break;
        }
        t = end;  // the run's end event
        if (oom) {
            rec(o.hl, o.hh, t, (j << 16) | (K_OOM << 12) | ev_lo);
            rec(o.hl, o.hh, t, (j << 16) | (K_FAILED << 12) | ev_lo);
            o.K2 += 1u << 16;
            o.K3 += 1u << 16;
        } else {
            rec(o.hl, o.hh, t, (j << 16) | (K_COMPLETE << 12) | ev_lo);
            if (lane == 0) o.acc += t;
        }
    }
    o.makespan = t;
    return o;
}

// Scheme A, schedule_by_group (reading R38): jobs are grouped by the memory level of their tight
// fit, groups run in ascending order on the level's homogeneous layout (geometry scheme_a_layouts), job k of a
// group goes to slice k mod #slices (static round robin in ascending start) and each slice runs its jobs in order;
// the GPU is reconfigured (LAYOUT record) only when a group has drained; OOM'd / preempted jobs join the tail of
// their new group. GL[l * cap + i] = i-th job of group l; lane l holds that group's length.
template <int GW, bool WIDE>
__device__ __forceinline__ TraceOut scheme_a_trace(const DevGeom& G, const Grp<GW>& g, uint32_t n,
                                                   const JobStore<WIDE>& J, uint16_t* GL, uint32_t cap, bool er,
                                                   bool fold, bool wave, uint32_t reconfig, uint32_t full_mem) {
    const uint32_t lane = g.gl;
    constexpr uint32_t kNone = 0xFFFFFFFFu;
    TraceOut o;
    o.K0 = o.K1 = o.K2 = o.K3 = 0;
    o.acc = 0;
    o.hl = (uint32_t)kFnvOffset;
    o.hh = (uint32_t)(kFnvOffset >> 32);
    uint32_t t = 0, glen = 0;
    // ---- t = 0: sorted_by_mig_group (REJECT records in queue order for jobs no profile holds) ----
    for (uint32_t c = 0; c < n; c += GW) {
        const uint32_t j = c + lane;
        const uint32_t need = j < n ? J.need(j) : 0xFEu;
        uint32_t rm = g.ballot(need == 0xFFu);
        while (rm) {
            const uint32_t k = (uint32_t)__ffs(rm) - 1u;
            rm &= rm - 1u;
            rec(o.hl, o.hh, t, ((c + k) << 16) | (K_REJECT << 12) | 0xFF0u);
            o.K2 += 1u;
        }
        const uint32_t lv = need < 0xFEu ? G.level[need] : 0xFFu;
        for (uint32_t l = 0; l < G.n_levels; ++l) {
            const uint32_t m = g.ballot(lv == l);
            if (!m) continue;
            const uint32_t b = g.shfl(glen, l);
            if (lv == l) GL[l * cap + b + __popc(m & ((1u << lane) - 1u))] = (uint16_t)j;
            if (lane == l) glen += __popc(m);
        }
    }
    g.sync();
    uint32_t cur = kNone, ii = 0, iend = 0, ijk = 0, nxt = 0, SM = 0, BM = 0, ns = 0, ready = 0;

    auto dispatch = [&]() {  // idle slices take their next job, ascending start
        const uint32_t len = g.shfl(glen, cur);
        uint32_t m = g.ballot((ii & kValid) && !(ii & kBusy) && nxt < len);
        while (m) {
            const uint32_t s = (uint32_t)__ffs(m) - 1u;
            m &= m - 1u;
            const uint32_t j = GL[cur * cap + g.shfl(nxt, s)];
            const uint32_t si = g.shfl(ii, s);
            rec(o.hl, o.hh, t, (j << 16) | (K_PLACE_GROUP << 12) | (s << 8) | (((si >> 20) & 0xFu) << 4));
            o.K0 += 1u;
            const uint32_t lev = si & 0xFu;
            uint32_t T, ticks, fe, pred, conv, phys;
            J.run_info(G, j, lev, T, ticks, fe, pred, conv, phys);
            if (wave) ticks = wave_ticks(G, ticks, J.warps(j), (si >> 20) & 0xFu);
            const uint32_t rs = t < ready ? t + reconfig : t;  // first run on a freshly created slice
            const uint32_t cap_m = G.level_mem[lev];
            uint32_t i_pre = 0xFFFFFFFFu;
            if (er && conv > 0 && pred > cap_m && cap_m < full_mem) i_pre = conv;
            uint32_t end, ek;
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
            if (lane == s) {
                ii |= kBusy;
                iend = end;
                ijk = j | (ek << 16);
                nxt += ns;
            }
            BM |= ((si >> 8) & 0xFFu) << s;
            acc_run(o.acc, lane, (uint64_t)((si >> 4) & 0xFu) * (end - rs), J.run_mem(j, phys, lev, ek, end - rs, ticks),
                    ek ? end - rs : 0u);
        }
    };
    auto next_group = [&]() -> bool {  // set_homogeneous_slices(next non-empty group)
        const uint32_t m = g.ballot(lane < G.n_levels && (cur == kNone || lane > cur) && glen > 0);
        if (!m) return false;
        const uint32_t l = (uint32_t)__ffs(m) - 1u;
        const uint32_t nd = __popc(SM);
        rec(o.hl, o.hh, t, (0xFFFFu << 16) | (K_LAYOUT << 12) | (l << 4) | nd);
        o.K1 += nd;
        ii = 0;
        SM = 0;
        ns = G.n_alay[l];
        for (uint32_t k = 0; k < ns; ++k) {
            const uint32_t e = G.alay[l][k], st = e & 0xFFu;
            if (lane == st) {
                ii = kValid | G.pinfo[e >> 8];
                nxt = k;
            }
            SM |= 1u << st;
        }
        o.K0 += ns << 16;
        ready = t + reconfig;
        cur = l;
        return true;
    };
    auto step = [&]() {
        if (cur != kNone) dispatch();
        for (;;) {
            if (cur != kNone) {
                const uint32_t len = g.shfl(glen, cur);
                if (BM || g.ballot((ii & kValid) && nxt < len)) break;  // the group has not drained
            }
            if (!next_group()) break;
            dispatch();
        }
    };

    step();
    for (;;) {
        const uint32_t mine = (ii & kBusy) ? iend : 0xFFFFFFFFu;
        const uint32_t tn = g.min(mine);
        if (tn == 0xFFFFFFFFu) break;
        t = tn;
        uint32_t evm = g.ballot(mine == t);
        do {
            uint32_t s;
            if ((evm & (evm - 1u)) == 0u) {
                s = (uint32_t)__ffs(evm) - 1u;
            } else {  // COMPLETE < OOM < PREEMPT, then job id (R28)
                const uint32_t key = ((evm >> lane) & 1u) ? ijk : 0xFFFFFFFFu;
                const uint32_t km = g.min(key);
                s = (uint32_t)__ffs(g.ballot(key == km)) - 1u;
            }
            evm &= ~(1u << s);
            const uint32_t si = g.shfl(ii, s);
            const uint32_t sjk = g.shfl(ijk, s);
            const uint32_t job = sjk & 0xFFFFu, ek = sjk >> 16;
            const uint32_t lo = (job << 16) | (s << 8) | (((si >> 20) & 0xFu) << 4);
            uint32_t req = 0;
            if (ek == 0) {
                rec(o.hl, o.hh, t, lo | (K_COMPLETE << 12));
                if (lane == 0) o.acc += t;
            } else if (ek == 1) {
                rec(o.hl, o.hh, t, lo | (K_OOM << 12));
                const uint32_t nl = G.level_next[si & 0xFu];
                o.K2 += 1u << 16;
                if (nl == 0) {
                    rec(o.hl, o.hh, t, lo | (K_FAILED << 12));
                    o.K3 += 1u << 16;
                } else {
                    req = nl;
                }
            } else {
                rec(o.hl, o.hh, t, lo | (K_PREEMPT << 12));
                o.K3 += 1u;
                req = min(J.pred(job), full_mem);
            }
            if (req) {  // the tail of the job's new (larger) group
                const uint32_t need = tight_fit_lane(G, req, J.warps(job), fold);
                if (need == 0xFFu) {
                    rec(o.hl, o.hh, t, (job << 16) | (K_REJECT << 12) | 0xFF0u);
                    o.K2 += 1u;
                } else {
                    const uint32_t lv = G.level[need];
                    const uint32_t b = g.shfl(glen, lv);
                    g.sync();
                    if (lane == 0) {
                        J.set_need(job, need);
                        GL[lv * cap + b] = (uint16_t)job;
                    }
                    g.sync();
                    if (lane == lv) ++glen;
                }
            }
            BM &= ~(((si >> 8) & 0xFFu) << s);
            if (lane == s) ii &= ~kBusy;
        } while (evm);
        step();
    }
    o.makespan = t;
    return o;
}

// One trace under one policy kind (Alg. 4 PAPER.md:601-617 + the partition manager).
template <int KIND, int GW, bool WIDE>
__device__ __forceinline__ TraceOut simulate_trace(const DevGeom& G, const Grp<GW>& g, uint32_t n,
                                                   const JobStore<WIDE>& J, uint16_t* ring, uint32_t ring_cap,
                                                   bool er, bool fold, bool wave, uint32_t reconfig,
                                                   uint32_t full_mem) {
    const uint32_t lane = g.gl;
    if constexpr (KIND == MIG_BASELINE) {
        return baseline_trace<WIDE>(G, n, J, g.gl);
    }
    uint32_t ii = 0, iend = 0, ijk = 0;  // lane-resident instance (slot = lane)
    uint32_t occ = 0, SM = 0, EM = 0, BM = 0;
    if (KIND == MIG_BASELINE) {
        const uint32_t fp = G.full_prof;
        if (lane == 0) ii = kValid | G.pinfo[fp];
        occ = G.lenmask[fp];
    } else if (KIND == MIG_STATIC) {
        for (uint32_t i = 0; i < G.n_layout; ++i) {
            const uint32_t p = G.layout_prof[i], s = G.layout_start[i];
            if (lane == s) ii = kValid | G.pinfo[p];
            occ |= G.lenmask[p] << s;
        }
    }
    TraceOut o;
    o.K0 = o.K1 = o.K2 = o.K3 = 0;
    o.acc = 0;
    o.hl = (uint32_t)kFnvOffset;
    o.hh = (uint32_t)(kFnvOffset >> 32);
    // queue = jobs[qh..n) ++ requeued jobs (tail, R13): a u16 ring (WIDE) or a list linked through the staged
    // records (NARROW; rh = head, rn = tail, 0xFFFF = empty)
    constexpr uint32_t kNone = 0xFFFFu;
    uint32_t t = 0, qh = 0, rh = WIDE ? 0u : kNone, rn = WIDE ? 0u : kNone;

    for (;;) {
        // ---------------- scheduler pass at tick t (head-of-line; wake on every event tick, R9) ----------------
        while (qh < n || (WIDE ? rn != 0 : rh != kNone)) {
            const uint32_t j = qh < n ? qh : (WIDE ? (uint32_t)ring[rh] : rh);
            const uint32_t need = J.need(j);
            const uint32_t jsh = j << 16;
            if (need == 0xFFu) {  // no profile can ever hold the job: REJECT
                rec(o.hl, o.hh, t, jsh | (K_REJECT << 12) | 0xFF0u);
                o.K2 += 1u;
            } else {
                const uint32_t pn = G.pinfo[need];
                const uint32_t nlev = pn & 0xFu, ncomp = (pn >> 4) & 0xFu;
                uint32_t s = 0, si = 0, kd = 0, nd = 0;
                bool created = false;
                if (KIND == MIG_BASELINE) {  // one job at a time on the whole GPU
                    if (BM) {
                        rec(o.hl, o.hh, t, jsh | (K_WAIT << 12) | 0xF00u | (need << 4));
                        o.K1 += 1u << 16;
                        break;
                    }
                    si = g.shfl(ii, 0);
                    kd = K_PLACE_BASELINE;
                } else if (KIND == MIG_STATIC) {  // smallest idle fitting layout slice, tie -> highest start (R11)
                    const uint32_t ilev = ii & 0xFu;
                    const bool cand = (ii & kValid) && ilev >= nlev && ((ii >> 4) & 0xFu) >= ncomp;
                    const uint32_t key = (cand && !(ii & kBusy)) ? (((15u - ilev) << 5) | lane) + 1u : 0u;
                    const uint32_t km = g.max(key);
                    if (!km) {
                        if (g.ballot(cand)) {
                            rec(o.hl, o.hh, t, jsh | (K_WAIT << 12) | 0xF00u | (need << 4));
                            o.K1 += 1u << 16;
                            break;
                        }
                        rec(o.hl, o.hh, t, jsh | (K_REJECT << 12) | 0xF00u | (need << 4));
                        o.K2 += 1u;
                        goto pop;
                    }
                    s = (km - 1u) & 31u;
                    si = g.shfl(ii, s);
                    kd = K_PLACE_STATIC;
                } else {
                    if (KIND == MIG_FUSION_FISSION) {  // an idle slice that tightly fits (R7)
                        const bool cand = (ii >> 30) == 2u && (ii & 0xFu) == nlev && ((ii >> 4) & 0xFu) >= ncomp;
                        const uint32_t m = g.ballot(cand);
                        if (m) {
                            s = 31u - __clz(m);
                            si = g.shfl(ii, s);
                            kd = K_REUSE;
                        }
                    }
                    if (!kd) {
                        // Alg. 2: C = legal placements of the tight profile; argmax fcr; tie -> highest start
                        const uint32_t pl = G.place[need][lane & 7u];
                        const uint32_t qm = pl >> 8;
                        const uint32_t score =
                            (pl && !(occ & qm)) ? ((uint32_t)G.fcr[occ | qm] << 8) | (pl & 0xFFu) : 0u;
                        const uint32_t best = g.max(score);
                        const uint32_t nlen = (pn >> 16) & 0xFu;
                        if (best) {
                            s = best & 0xFFu;
                            kd = K_ALLOC;
                        } else if (KIND == MIG_FUSION_FISSION) {
                            // fusion / fission: destroy the idle instances placement k overlaps (none busy, >= 1),
                            // best (fcr(result), -#destroyed, start) (R8)
                            uint32_t sc = 0;
                            if (pl && !(qm & BM) && (qm & occ)) {
                                const uint32_t lo = pl & 0xFFu;
                                const uint32_t rm = overlap_extent(occ, SM, EM, lo, lo + nlen - 1u);
                                sc = ((uint32_t)G.fcr[(occ & ~rm) | qm] << 16) | ((15u - __popc(SM & rm)) << 8) | lo;
                            }
                            const uint32_t bs = g.max(sc);
                            if (bs) {
                                s = bs & 0xFFu;
                                nd = 15u - ((bs >> 8) & 0xFFu);
                                const uint32_t rm = overlap_extent(occ, SM, EM, s, s + nlen - 1u);
                                if ((SM & rm) >> lane & 1u) ii = 0;  // destroy (all idle)
                                occ &= ~rm;
                                SM &= ~rm;
                                EM &= ~rm;
                                kd = K_RECONF;
                            }
                        }
                        if (!kd) {  // sleep() until a running job finishes
                            rec(o.hl, o.hh, t, jsh | (K_WAIT << 12) | 0xF00u | (need << 4));
                            o.K1 += 1u << 16;
                            break;
                        }
                        // create the instance (try_new_mig_slice)
                        created = true;
                        occ |= ((pn >> 8) & 0xFFu) << s;
                        if (KIND == MIG_FUSION_FISSION) {
                            SM |= 1u << s;
                            EM |= 1u << (s + nlen - 1u);
                        }
                        si = kValid | pn;
                        if (lane == s) ii = si;
                    }
                }
                // the decision record, then start the run
                const uint32_t prof = (si >> 20) & 0xFu;
                rec(o.hl, o.hh, t, jsh | (kd << 12) | (s << 8) | (prof << 4) | nd);
                o.K0 += created ? 0x10001u : 1u;
                o.K1 += nd;
                const uint32_t lev = si & 0xFu;
                uint32_t T, ticks, fe, pred, conv, phys;  // conv = 0 unless a converged DYNAMIC forecast
                J.run_info(G, j, lev, T, ticks, fe, pred, conv, phys);
                if (wave) ticks = wave_ticks(G, ticks, J.warps(j), (si >> 20) & 0xFu);
                const uint32_t rs = t + (created ? reconfig : 0u);
                const uint32_t cap = G.level_mem[lev];
                uint32_t i_pre = 0xFFFFFFFFu;
                if (KIND != MIG_BASELINE && er && conv > 0 && pred > cap && cap < full_mem) i_pre = conv;
                uint32_t end, ek;
                if (fe <= min(T, i_pre)) {  // OOM > COMPLETE > PREEMPT in one iteration (R29); NEVER = 0xFFFF > T
                    ek = 1;
                    end = rs + fe * ticks;
                } else if (i_pre < T) {
                    ek = 2;
                    end = rs + i_pre * ticks;
                } else {
                    ek = 0;
                    end = rs + T * ticks;
                }
                if (lane == s) {
                    ii |= kBusy;
                    iend = end;
                    ijk = j | (ek << 16);
                }
                BM |= ((si >> 8) & 0xFFu) << s;
                acc_run(o.acc, lane, (uint64_t)((si >> 4) & 0xFu) * (end - rs),
                        J.run_mem(j, phys, lev, ek, end - rs, ticks), ek ? end - rs : 0u);
            }
        pop:
            if (qh < n) {
                ++qh;
            } else if (WIDE) {
                rh = rh + 1 == ring_cap ? 0 : rh + 1;
                --rn;
            } else {
                rh = J.next(rh);
                if (rh == kNone) rn = kNone;
            }
        }
        // ---------------- next event: min end tick over running instances ----------------
        const uint32_t mine = (ii & kBusy) ? iend : 0xFFFFFFFFu;
        const uint32_t tn = g.min(mine);
        if (tn == 0xFFFFFFFFu) break;
        t = tn;
        uint32_t evm = g.ballot(mine == t);
        do {
            uint32_t s;
            if ((evm & (evm - 1u)) == 0u) {
                s = (uint32_t)__ffs(evm) - 1u;
            } else {  // several events at one tick: COMPLETE < OOM < PREEMPT, then job id (R28)
                const uint32_t key = ((evm >> lane) & 1u) ? ijk : 0xFFFFFFFFu;  // kind << 16 | job
                const uint32_t km = g.min(key);
                s = (uint32_t)__ffs(g.ballot(key == km)) - 1u;
            }
            evm &= ~(1u << s);
            const uint32_t si = g.shfl(ii, s);
            const uint32_t sjk = g.shfl(ijk, s);
            const uint32_t job = sjk & 0xFFFFu, ek = sjk >> 16;
            const uint32_t lo = (job << 16) | (s << 8) | (((si >> 20) & 0xFu) << 4);
            uint32_t req = 0;
            if (ek == 0) {
                rec(o.hl, o.hh, t, lo | (K_COMPLETE << 12));
                if (lane == 0) o.acc += t;
            } else if (ek == 1) {  // OOM: next larger slice (R14) or FAILED on the whole GPU
                rec(o.hl, o.hh, t, lo | (K_OOM << 12));
                const uint32_t nl = G.level_next[si & 0xFu];
                o.K2 += 1u << 16;
                if (nl == 0) {
                    rec(o.hl, o.hh, t, lo | (K_FAILED << 12));
                    o.K3 += 1u << 16;
                } else {
                    req = nl;
                }
            } else {  // PREEMPT: restart on the slice meeting the forecast (R25)
                rec(o.hl, o.hh, t, lo | (K_PREEMPT << 12));
                o.K3 += 1u;
                req = min(J.pred(job), full_mem);
            }
            if (req) {  // back to the queue tail (R13) with the new tight fit
                const uint32_t need = tight_fit_lane(G, req, J.warps(job), fold);
                g.sync();
                if (lane == 0) {
                    J.set_need(job, need);
                    if (WIDE) {
                        uint32_t pos = rh + rn;
                        if (pos >= ring_cap) pos -= ring_cap;
                        ring[pos] = (uint16_t)job;
                    } else {
                        J.set_next(job, kNone);
                        if (rn != kNone) J.set_next(rn, job);
                    }
                }
                g.sync();
                if (WIDE) {
                    ++rn;
                } else {
                    if (rn == kNone) rh = job;
                    rn = job;
                }
            }
            const uint32_t ext = ((si >> 8) & 0xFFu) << s;
            BM &= ~ext;
            if (KIND == MIG_DYNAMIC) {  // free on completion (R10)
                if (lane == s) ii = 0;
                occ &= ~ext;
                o.K1 += 1u;
            } else if (lane == s) {
                ii &= ~kBusy;
            }
        } while (evm);
    }
    o.makespan = t;
    return o;
}

template <int GW, bool WIDE, int WARPS, bool SA>
__global__ void __launch_bounds__(WARPS * 32, 32 / WARPS) k_simulate(const DevGeom* __restrict__ Gg, const SimParams P) {
    extern __shared__ __align__(16) uint8_t smem[];
    DevGeom& G = *reinterpret_cast<DevGeom*>(smem);
    mig_policy* s_pol = reinterpret_cast<mig_policy*>(smem + kGeomBytes);
    unsigned long long* s_tot = reinterpret_cast<unsigned long long*>(smem + kGeomBytes + kPolBytes);
    const Grp<GW> g(threadIdx.x & 31u);
    const uint32_t lane = g.gl, group = threadIdx.x / GW;
    const uint32_t gl_bytes = P.scheme_a ? ((kMaxLevels * P.max_jobs * 2u + 15u) & ~15u) : 0u;
    const uint32_t per_group =
        (WIDE ? P.max_jobs * 32u + ((P.max_jobs * 2u + 15u) & ~15u) : P.max_jobs * 16u) + gl_bytes;
    uint8_t* wb = smem + kGeomBytes + kPolBytes + kTotBytes + group * per_group;
    uint16_t* GL = reinterpret_cast<uint16_t*>(wb + per_group - gl_bytes);  // Scheme A group lists
    uint4* jobA = reinterpret_cast<uint4*>(wb);
    uint4* jobB = WIDE ? jobA + P.max_jobs : nullptr;
    uint16_t* ring = WIDE ? reinterpret_cast<uint16_t*>(jobA + P.max_jobs * 2u) : nullptr;  // requeue FIFO (WIDE)

    {
        const uint32_t* src = reinterpret_cast<const uint32_t*>(Gg);
        uint32_t* dst = reinterpret_cast<uint32_t*>(smem);
        for (uint32_t i = threadIdx.x; i < sizeof(DevGeom) / 4; i += blockDim.x) dst[i] = __ldg(src + i);
        if (threadIdx.x == 0) {
#pragma unroll
            for (int k = 0; k < kMaxPolicies; ++k) s_pol[k] = P.pol[k];
        }
        for (uint32_t i = threadIdx.x; i < kMaxPolicies * kTotFields; i += blockDim.x) s_tot[i] = 0;
    }
    __syncthreads();
    const uint32_t full_mem = G.full_mem;

    const uint64_t j_base = P.off[0];
    for (;;) {
        unsigned long long tr = 0;
        if (lane == 0) tr = atomicAdd(P.counter, 1ull);
        tr = g.shfl64(tr, 0);
        if (tr >= P.n_traces) break;
        const uint64_t j0 = P.off[tr] - j_base;
        const uint64_t n64 = P.off[tr + 1] - P.off[tr];
        uint32_t err = 0;
        uint32_t n = (uint32_t)n64;
        if (n64 > P.max_jobs) {
            err |= (uint32_t)MIG_ERR_TRACE_TOO_LONG;
            n = 0;
        }
        // ---- a1/a2: stage the trace (128-bit coalesced loads) and the per-job estimates ----
        for (uint32_t j = lane; j < n; j += GW) {
            const uint4 r = __ldg(P.jobs + j0 + j);
            const uint4 e = P.ext ? __ldg(P.ext + j0 + j) : make_uint4(0, 0, 0, 0);
            const uint32_t cls = (r.z >> 16) & 0xFFu, T = r.z & 0xFFFFu;
            if (cls > 2 || T > 4096) err |= (uint32_t)MIG_ERR_BAD_RECORD;
            uint4 A, Bv;
            A.x = T | (cls << 16);
            A.y = r.w;
            if (cls == kClassDynamic) {
                const uint4* es = reinterpret_cast<const uint4*>(P.est + j0 + j);
                const uint4 e0 = __ldg(es);
                if (WIDE) {
                    const uint4 e1 = __ldg(es + 1);
                    A.z = e0.x;  // req0 (smallest slice, R16)
                    A.w = e.y;
                    Bv = make_uint4(e0.y, (e0.z & 0xFFFFu) | (e0.w << 16), (e0.w >> 16) | (e1.x << 16),
                                    (e1.x >> 16) | (e1.y << 16));
                } else {
                    A.z = e0.y;             // pred
                    A.w = e0.z & 0xFFFFu;   // conv
                }
            } else {
                // physical footprint true + ws + ctx; exceeds level l at iteration 1 or never (R12)
                const uint64_t phys64 = (uint64_t)r.y + e.x + P.ctx;
                const uint32_t phys = phys64 > 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)phys64;
                if (WIDE) {
                    A.z = r.x + e.x + P.ctx;  // req0 = est + ws + ctx
                    A.w = e.y;
                    uint32_t fe[5];
#pragma unroll
                    for (int l = 0; l < kMaxLevels; ++l)
                        fe[l] = (l < (int)G.n_levels && T >= 1 && phys > G.level_mem[l]) ? 1u : kNever;
                    Bv = make_uint4(phys, fe[0] << 16, fe[1] | (fe[2] << 16), fe[3] | (fe[4] << 16));
                } else {
                    A.z = phys;
                    A.w = 0;  // conv = 0; high half: requeue link
                }
            }
            jobA[j] = A;
            if (WIDE) jobB[j] = Bv;
        }
        err = g.bor(err);

        for (uint32_t p = 0; p < P.n_pol; ++p) {
            const mig_policy& pol = s_pol[p];
            const uint32_t kind = pol.kind;
            const bool fold = (pol.flags & MIG_WARP_FOLD) != 0;
            const bool er = (pol.flags & MIG_EARLY_RESTART) != 0;
            const bool wave = (pol.flags & MIG_WAVE_TIME) != 0;
            g.sync();
            for (uint32_t j = lane; j < n; j += GW) {
                const uint4 A = jobA[j];
                uint32_t req0, warps;
                if (WIDE) {
                    req0 = A.z;
                    warps = A.w;
                } else {  // re-read the record: req0 = est + ws + ctx, or the smallest slice (DYNAMIC, R16)
                    const uint4 r = __ldg(P.jobs + j0 + j);
                    const uint4 e = P.ext ? __ldg(P.ext + j0 + j) : make_uint4(0, 0, 0, 0);
                    req0 = ((r.z >> 16) & 0xFFu) == kClassDynamic ? G.mem[0] : r.x + e.x + P.ctx;
                    warps = e.y;
                }
                jobA[j].x = (A.x & 0x00FFFFFFu) | (tight_fit_lane(G, req0, warps, fold) << 24);
            }
            g.sync();
            const JobStore<WIDE> J{jobA, jobB, P.jobs + j0, P.ext ? P.ext + j0 : nullptr, P.est + j0, P.ctx};
            TraceOut o;
            if (SA)  // separate instantiation: Scheme A's state does not raise the Scheme B loop's registers
                o = scheme_a_trace<GW, WIDE>(G, g, n, J, GL, P.max_jobs, er, fold, wave, pol.reconfig_ticks, full_mem);
            else if (kind == MIG_FUSION_FISSION)
                o = simulate_trace<MIG_FUSION_FISSION, GW, WIDE>(G, g, n, J, ring, P.ring_cap, er, fold, wave,
                                                           pol.reconfig_ticks, full_mem);
            else if (kind == MIG_DYNAMIC)
                o = simulate_trace<MIG_DYNAMIC, GW, WIDE>(G, g, n, J, ring, P.ring_cap, er, fold, wave,
                                                    pol.reconfig_ticks, full_mem);
            else if (kind == MIG_STATIC)
                o = simulate_trace<MIG_STATIC, GW, WIDE>(G, g, n, J, ring, P.ring_cap, er, fold, wave,
                                                   pol.reconfig_ticks, full_mem);
            else
                o = simulate_trace<MIG_BASELINE, GW, WIDE>(G, g, n, J, ring, P.ring_cap, er, fold, wave,
                                                     pol.reconfig_ticks, full_mem);
            // ---- a11: per-trace result (80 B, five 128-bit stores from lanes 0-4) ----
            const uint32_t placements = o.K0 & 0xFFFFu, creates = o.K0 >> 16, destroys = o.K1 & 0xFFFFu,
                           waits = o.K1 >> 16, rejected = o.K2 & 0xFFFFu, ooms = o.K2 >> 16,
                           preempts = o.K3 & 0xFFFFu, failed = o.K3 >> 16;
            const uint32_t completed = n - rejected - failed, restarts = ooms - failed + preempts;
            const uint64_t turn = g.shfl64(o.acc, 0), busy = g.shfl64(o.acc, 1), memt = g.shfl64(o.acc, 2),
                           wasted = g.shfl64(o.acc, 3);
            const uint64_t energy = (uint64_t)pol.idle_w * o.makespan + (uint64_t)pol.w_per_slice * busy;
            if (P.out && lane < 6) {
                uint4 v;
                if (lane == 0) v = make_uint4(o.makespan, n, completed, rejected);
                else if (lane == 1) v = make_uint4(failed, ooms, preempts, restarts);
                else if (lane == 2) v = make_uint4(placements, waits, creates, destroys);
                else if (lane == 3) v = make_uint4((uint32_t)energy, (uint32_t)(energy >> 32), (uint32_t)turn,
                                                   (uint32_t)(turn >> 32));
                else if (lane == 4) v = make_uint4((uint32_t)busy, (uint32_t)(busy >> 32), o.hl, o.hh);
                else v = make_uint4((uint32_t)memt, (uint32_t)(memt >> 32), (uint32_t)wasted,
                                    (uint32_t)(wasted >> 32));
                reinterpret_cast<uint4*>(P.out + tr * P.n_pol_all + P.pol_idx[p])[lane] = v;
            }
            // ---- a12: per-policy totals (shared-memory atomics, flushed once per CTA) ----
            for (uint32_t f = lane; f < 21; f += GW) {
                uint64_t v;
                switch (f) {
                    case 0: v = 1; break;
                    case 1: v = n; break;
                    case 2: v = completed; break;
                    case 3: v = rejected; break;
                    case 4: v = failed; break;
                    case 5: v = ooms; break;
                    case 6: v = preempts; break;
                    case 7: v = restarts; break;
                    case 8: v = placements; break;
                    case 9: v = waits; break;
                    case 10: v = creates; break;
                    case 11: v = destroys; break;
                    case 12:
                    case 13: v = o.makespan; break;
                    case 14: v = energy; break;
                    case 15: v = turn; break;
                    case 16: v = busy; break;
                    case 17: v = ((uint64_t)o.hh << 32) | o.hl; break;
                    case 18: v = memt; break;
                    case 19: v = wasted; break;
                    default: v = err; break;
                }
                if (f == 13) atomicMax(&s_tot[p * kTotFields + 13], (unsigned long long)v);
                else if (f == 20) { if (v) atomicOr(&s_tot[p * kTotFields + 20], (unsigned long long)v); }
                else atomicAdd(&s_tot[p * kTotFields + f], (unsigned long long)v);
            }
        }
    }
    __syncthreads();
    if (P.totals && blockIdx.x == 0 && threadIdx.x < P.n_pol && P.est_err && *P.est_err)
        atomicOr(reinterpret_cast<unsigned long long*>(P.totals + P.pol_idx[threadIdx.x]) + 20, *P.est_err);
    if (P.totals) {
        for (uint32_t i = threadIdx.x; i < P.n_pol * kTotFields; i += blockDim.x) {
            const uint32_t f = i % kTotFields;
            unsigned long long* dst =
                reinterpret_cast<unsigned long long*>(P.totals + P.pol_idx[i / kTotFields]) + f;
            if (f == 13) atomicMax(dst, s_tot[i]);
            else if (f == 20) { if (s_tot[i]) atomicOr(dst, s_tot[i]); }
            else if (f < 20) atomicAdd(dst, s_tot[i]);
        }
    }
}

constexpr int warps_per_cta(bool wide) { return wide ? 4 : 8; }

size_t simulate_smem_bytes(uint32_t max_jobs, int gw, bool wide, bool scheme_a) {
    const size_t per_group = (wide ? (size_t)max_jobs * 32u + ((max_jobs * 2u + 15u) & ~15u) : (size_t)max_jobs * 16u) +
                             (scheme_a ? ((kMaxLevels * max_jobs * 2u + 15u) & ~15u) : 0u);
    return kGeomBytes + kPolBytes + kTotBytes + (size_t)(warps_per_cta(wide) * 32 / gw) * per_group;
}

template <int GW, bool WIDE, bool SA>
static cudaError_t launch_gw(const DevGeom* Gdev, const SimParams& P, uint64_t n_traces, int sm_count,
                             cudaStream_t stream) {
    constexpr int kW = warps_per_cta(WIDE);
    const size_t smem = simulate_smem_bytes(P.max_jobs, GW, WIDE, SA);
    cudaError_t e =
        cudaFuncSetAttribute(k_simulate<GW, WIDE, kW, SA>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_simulate<GW, WIDE, kW, SA>, kW * 32, smem);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    const uint64_t groups = (uint64_t)kW * 32 / GW;
    uint64_t want = (n_traces + groups - 1) / groups;
    uint64_t blocks = (uint64_t)per_sm * sm_count;
    if (want < blocks) blocks = want;
    if (blocks < 1) blocks = 1;
    k_simulate<GW, WIDE, kW, SA><<<(unsigned)blocks, kW * 32, smem, stream>>>(Gdev, P);
    return cudaGetLastError();
}

// Lanes per trace: 8 (four traces per warp) unless MIG_LANES_PER_TRACE=32 (one trace per warp) or the staged
// traces would not fit shared memory four to a warp.
int simulate_group_width(uint32_t max_jobs, bool scheme_a) {
    static int forced = -1;
    if (forced < 0) {
        const char* env = getenv("MIG_LANES_PER_TRACE");
        forced = env ? atoi(env) : 0;
    }
    if (forced == 32 || forced == 8) return forced;
    return simulate_smem_bytes(max_jobs, 8, false, scheme_a) <= 200 * 1024 ? 8 : 32;
}

// Staging layout: 32 B/job for short traces (everything on chip), 16 B/job for long ones (occupancy).
bool simulate_wide_layout(uint32_t max_jobs) {
    static int forced = -1;
    if (forced < 0) {
        const char* env = getenv("MIG_JOB_LAYOUT");
        forced = env ? (strcmp(env, "wide") == 0 ? 1 : strcmp(env, "narrow") == 0 ? 2 : 0) : 0;
    }
    if (forced) return forced == 1;
    return max_jobs <= 32;
}

template <bool SA>
static cudaError_t launch_variant(const DevGeom* Gdev, const SimParams& P, const mig_traces& tr, int sm_count,
                                  cudaStream_t stream) {
    const bool wide = simulate_wide_layout(tr.max_jobs);
    if (simulate_group_width(tr.max_jobs, SA) == 8)
        return wide ? launch_gw<8, true, SA>(Gdev, P, tr.n_traces, sm_count, stream)
                    : launch_gw<8, false, SA>(Gdev, P, tr.n_traces, sm_count, stream);
    return wide ? launch_gw<32, true, SA>(Gdev, P, tr.n_traces, sm_count, stream)
                : launch_gw<32, false, SA>(Gdev, P, tr.n_traces, sm_count, stream);
}

uint64_t simulate_lane_grid(uint64_t n_traces, int sm_count);
uint32_t simulate_lane_threads();
uint32_t simulate_lane_partials();
size_t trace_order_scratch_bytes(uint64_t n_traces);  // trace_order.cu
cudaError_t launch_trace_order(const mig_traces& tr, const DevGeom* Gh, uint32_t ctx, void* buf, bool force,
                               int sm_count, cudaStream_t s);
cudaError_t launch_simulate_lane(const DevGeom* Gdev, const mig_traces& tr, const mig_policy& pol, uint32_t pol_idx,
                                 uint32_t n_pol_all, const mig_job_estimate* est, mig_trace_result* out,
                                 mig_policy_totals* totals, unsigned long long* counter,
                                 const unsigned long long* est_err, uint16_t* ring, uint64_t blocks,
                                 const uint16_t* sid, const uint32_t* a7, uint32_t n_a7,
                                 uint4* pc, unsigned long long* part, int sm_count, cudaStream_t stream,
                                 const DevGeom* Gh, const uint32_t* order);

// Scheme B policies run one lane per trace (simulate_lane.cu) unless MIG_LANES_PER_TRACE selects the group kernel
// (8 or 32 lanes per trace).
bool simulate_use_lane() {
    static int forced = -1;
    if (forced < 0) {
        const char* env = getenv("MIG_LANES_PER_TRACE");
        forced = env ? atoi(env) : 1;
    }
    return forced == 1;
}

static int env_flag(const char* name, int dflt) {
    const char* v = getenv(name);
    return v ? atoi(v) : dflt;
}

// Policy launches on forked streams (launch_simulate): on unless MIG_CONCURRENT_POLICIES=0.
bool simulate_concurrent() {
    static int on = -1;
    if (on < 0) {
        const char* env = getenv("MIG_CONCURRENT_POLICIES");
        on = env ? atoi(env) != 0 : 1;
    }
    return on != 0;
}

// Up to `want` non-blocking side streams of device `dev` for the calling thread (created on first use, kept for the
// thread's lifetime). Per thread, so calls from different threads never share a side stream: no false dependency
// between them through the join event, and a thread capturing mig_simulate into a CUDA graph pulls only its own side
// stream into the capture.
namespace {
struct ThreadSideStreams {
    cudaStream_t s[64][kMaxPolicies] = {};
    uint32_t have[64] = {};
    ~ThreadSideStreams() {
        for (int d = 0; d < 64; ++d)
            for (uint32_t i = 0; i < have[d]; ++i) cudaStreamDestroy(s[d][i]);  // errors at process exit ignored
    }
};
thread_local ThreadSideStreams t_side;
}  // namespace

static uint32_t lane_side_streams(int dev, uint32_t want, cudaStream_t* out) {
    if (dev < 0 || dev >= 64) return 0;
    if (want > kMaxPolicies - 1) want = kMaxPolicies - 1;
    while (t_side.have[dev] < want) {
        if (cudaStreamCreateWithFlags(&t_side.s[dev][t_side.have[dev]], cudaStreamNonBlocking) != cudaSuccess) {
            cudaGetLastError();
            break;
        }
        ++t_side.have[dev];
    }
    const uint32_t n = t_side.have[dev] < want ? t_side.have[dev] : want;
    for (uint32_t i = 0; i < n; ++i) out[i] = t_side.s[dev][i];
    return n;
}

// Whether launch_simulate runs every policy on the lane kernels (which need no estimates for STATIC / MODEL jobs).
bool simulate_lane_path(uint32_t n_prof, const void* sid, const void* a7) {
    return simulate_use_lane() && n_prof <= 8 && sid && a7;
}

// counter: kSimCounters zeroed u64 trace counters ([0] group kernel Scheme B, [1] group kernel Scheme A,
// [2 + i] lane kernel, policy i).
cudaError_t launch_simulate(const DevGeom* Gdev, const mig_traces& tr, const mig_policy* pols, uint32_t n_pol,
                            const mig_job_estimate* est, mig_trace_result* out, mig_policy_totals* totals,
                            unsigned long long* counter, const unsigned long long* est_err, int sm_count,
                            cudaStream_t stream, uint32_t* launches, uint32_t n_prof, const uint16_t* sid,
                            const uint32_t* a7, uint32_t n_a7, const DevGeom* Gh) {
    SimParams P;
    memset(&P, 0, sizeof(P));
    P.jobs = (const uint4*)tr.jobs;
    P.ext = (const uint4*)tr.jobs_ext;
    P.off = tr.trace_off;
    P.est = est;
    P.n_traces = tr.n_traces;
    P.out = out;
    P.totals = totals;
    P.counter = counter;
    P.est_err = est_err;
    P.max_jobs = tr.max_jobs;
    P.ring_cap = tr.max_jobs;
    P.n_pol_all = n_pol;
    P.ctx = pols[0].ctx_mib;
    SimParams PA = P;  // Scheme A policies
    P.n_pol = PA.n_pol = 0;
    for (uint32_t i = 0; i < n_pol; ++i) {
        SimParams& Q = pols[i].kind == MIG_SCHEME_A ? PA : P;
        Q.pol_idx[Q.n_pol] = i;
        Q.pol[Q.n_pol++] = pols[i];
    }
    PA.scheme_a = 1;
    PA.counter = counter + 1;
    cudaError_t e = cudaSuccess;
    *launches = 0;
    // the lane kernel packs idle masks per profile in a u64 and takes fusion / fission from the host tables
    const bool lane = simulate_use_lane() && n_prof <= 8 && sid && a7;
    if (lane) {  // every policy, Scheme A included: one lane-kernel launch each
        // The policies' launches are independent (own trace counter, scratch, results column, totals row), so
        // they alternate between `stream` and one forked side stream: each launch's CTAs start on the SMs the
        // previous launch's tail leaves idle (persistent grids with per-lane work stealing end unevenly), while
        // at most two launches share the GPU (more streams mixed kernels of different residency on an SM and
        // ran slower, config 5). Fork / join by events keeps the call stream-ordered on `stream` (and capturable
        // in a CUDA graph). MIG_CONCURRENT_POLICIES=0 serialises every launch on `stream`.
        const uint64_t blocks = simulate_lane_grid(tr.n_traces, sm_count);
        const uint64_t stride = (uint64_t)tr.max_jobs * (PA.n_pol ? kMaxLevels : 1);  // Scheme A: group lists
        const size_t ring_elems = blocks * simulate_lane_threads() * stride;
        bool any_pc = false;  // PCIe contention (R39): per lane and slot run state
        for (uint32_t i = 0; i < n_pol; ++i) any_pc |= (pols[i].flags & MIG_PCIE_CONTENTION) != 0;
        const size_t pc_elems = any_pc ? blocks * simulate_lane_threads() * 8 * 2 : 0;
        int dev = 0;
        e = cudaGetDevice(&dev);
        if (e != cudaSuccess) return e;
        cudaStream_t side[kMaxPolicies] = {};
        const uint32_t n_side = (simulate_concurrent() && n_pol > 1) ? lane_side_streams(dev, 1u, side) : 0u;
        const uint32_t n_scr = n_side + 1;  // scratch sets: one per concurrently running launch
        // per scratch set (one per stream): requeue FIFOs / group lists (u16), then per-lane partial totals (u64)
        const size_t part_elems = blocks * simulate_lane_threads() * simulate_lane_partials();
        const size_t ring_bytes = (ring_elems * sizeof(uint16_t) + 255) & ~(size_t)255;
        const size_t set_bytes = ring_bytes + part_elems * sizeof(unsigned long long);
        char* scr = nullptr;
        e = mig_scratch_alloc((void**)&scr, n_scr * set_bytes, stream);
        if (e != cudaSuccess) return e;
        uint4* pc = nullptr;
        if (any_pc) {
            e = mig_scratch_alloc((void**)&pc, n_scr * pc_elems * sizeof(uint4), stream);
            if (e != cudaSuccess) {
                mig_scratch_free(scr, stream);
                return e;
            }
        }
        // the visit order of the traces (trace_order.cu): similar traces in neighbouring lanes, one pass for every
        // policy launch (a schedule only: results do not depend on it). Default: calls of at least 4096 traces
        // averaging at least 32 jobs (a lane's phases only matter over long queues: configs 3 and 4, 20 and 4 jobs
        // per trace, ran slower ordered), and the pass itself keeps trace order unless a quarter of the queues look
        // homogeneous (config 5's mixed queues ran slower ordered); MIG_TRACE_ORDER=0 keeps trace order, =2 orders
        // every call (tests)
        uint32_t* order = nullptr;
        const int ord = env_flag("MIG_TRACE_ORDER", 1);
        const bool long_queues = tr.n_jobs >= 32 * tr.n_traces;
        bool ff_kind = false;  // k_ff_lane visits the order (FUSION_FISSION / DYNAMIC on plain records)
        for (uint32_t i = 0; i < n_pol; ++i)
            ff_kind |= pols[i].kind == MIG_FUSION_FISSION || pols[i].kind == MIG_DYNAMIC;
        if (Gh && ord && ff_kind && !tr.jobs_ext && ((tr.n_traces >= 4096 && long_queues) || ord == 2) &&
            tr.n_traces < (1ull << 32)) {
            e = mig_scratch_alloc((void**)&order, trace_order_scratch_bytes(tr.n_traces), stream);
            if (e == cudaSuccess)
                e = (cudaError_t)mig_timed("sim_order", stream, [&](uint32_t* nl) {
                    if (nl) *nl = 3;
                    return (int)launch_trace_order(tr, Gh, pols[0].ctx_mib, order, ord == 2, sm_count, stream);
                });
            if (e != cudaSuccess) {
                if (order) mig_scratch_free(order, stream);
                mig_scratch_free(scr, stream);
                if (pc) mig_scratch_free(pc, stream);
                return e;
            }
            *launches += 3;
        }
        cudaEvent_t fork = nullptr, join[kMaxPolicies] = {};
        if (n_side) {
            e = cudaEventCreateWithFlags(&fork, cudaEventDisableTiming);
            if (e == cudaSuccess) e = cudaEventRecord(fork, stream);
        }
        // timing groups (mig_timing_enable): "~" marks launches on the side stream, whose events also span the
        // wait for the SMs of the launch before them
        static const char* kNames[2][5] = {{"sim_baseline", "sim_static", "sim_dynamic", "sim_ff", "sim_scheme_a"},
                                           {"sim_baseline~", "sim_static~", "sim_dynamic~", "sim_ff~", "sim_scheme_a~"}};
        for (uint32_t i = 0; i < n_pol && e == cudaSuccess; ++i) {
            const uint32_t k = n_side ? i % n_scr : 0u;  // stream / scratch set of policy i
            cudaStream_t st = k ? side[k - 1] : stream;
            if (k && i < n_scr) e = cudaStreamWaitEvent(st, fork, 0);
            if (e != cudaSuccess) break;
            e = (cudaError_t)mig_timed(kNames[k ? 1 : 0][pols[i].kind], st, [&](uint32_t* nl) {
                if (nl) *nl = 1;
                return (int)launch_simulate_lane(Gdev, tr, pols[i], i, n_pol, est, out, totals, counter + 2 + i,
                                                 est_err, reinterpret_cast<uint16_t*>(scr + k * set_bytes), blocks,
                                                 sid, a7, n_a7, pc ? pc + k * pc_elems : nullptr,
                                                 reinterpret_cast<unsigned long long*>(scr + k * set_bytes + ring_bytes),
                                                 sm_count, st, Gh, order);
            });
            ++*launches;
        }
        for (uint32_t k = 1; k < n_scr; ++k) {  // join: `stream` waits for every side stream's launches
            cudaError_t e2 = cudaEventCreateWithFlags(&join[k], cudaEventDisableTiming);
            if (e2 == cudaSuccess) e2 = cudaEventRecord(join[k], side[k - 1]);
            if (e2 == cudaSuccess) e2 = cudaStreamWaitEvent(stream, join[k], 0);
            if (e == cudaSuccess) e = e2;
            if (join[k]) cudaEventDestroy(join[k]);
        }
        if (fork) cudaEventDestroy(fork);
        if (order) mig_scratch_free(order, stream);
        mig_scratch_free(scr, stream);
        if (pc) mig_scratch_free(pc, stream);
        return e;
    }
    for (uint32_t i = 0; i < n_pol; ++i)  // the group kernel has no contention model and no arrival streams
        if ((pols[i].flags & MIG_PCIE_CONTENTION) || tr.arrival) return cudaErrorNotSupported;
    if (P.n_pol) {
        e = launch_variant<false>(Gdev, P, tr, sm_count, stream);
        if (e != cudaSuccess) return e;
        ++*launches;
    }
    if (PA.n_pol) {
        // est_err is OR-ed into every policy row of both launches (an OR is idempotent)
        e = launch_variant<true>(Gdev, PA, tr, sm_count, stream);
        if (e != cudaSuccess) return e;
        ++*launches;
    }
    return e;
}

}  // namespace mig
