// simulate_ff.cu — the two specialised lane kernels of the common cases (no warp folding / wave time, no arrival
// streams or PCIe contention): k_ff_lane (FUSION_FISSION, with or without early restart) and k_base_lane
// (BASELINE), SURVEY.md §8(a) rows a1, a4-a12 (a9, a10). Both take extension records (XR: the workspace field joins
// the estimate and the true footprint) as a template option. Same method, decision records, counters and results as
// the generic k_simulate_lane (simulate_lane.cu), which keeps every other case; launch_simulate_lane picks these when
// they apply (MIG_FF_FAST=0 disables them for A/B runs and parity of both paths).
#include <algorithm>

#include "lane_common.cuh"

namespace mig {

// ================================================================================================================
// k_ff_lane: the FUSION_FISSION launch of the common cases (no warp folding / wave time, no arrival streams or PCIe
// contention) written for the fewest issued instructions per step. XR: extension records (their workspace field is
// added to the record's estimate and true footprint when the record is fetched, R17); ER: MIG_EARLY_RESTART (a10,
// a DYNAMIC job whose converged forecast exceeds its slice is preempted at the convergence iteration
// and requeued for the forecast, R25). Same method, records, counters and results as k_simulate_lane
// <MIG_FUSION_FISSION> (parity-tested against the oracle by the same suites); what differs is the bookkeeping:
//  - the running instances' next events are 64-bit keys {end tick, kind, job, slot} in shared memory, so the next
//    event of a lane (R28: tick, then COMPLETE < OOM < PREEMPT, then job id) is one unrolled minimum over the 8
//    start slots, kept in a register (kmin) and refreshed only when an event retires; a tick's remaining events
//    and the move to the scheduler pass need no per-tick event mask or tie loop;
//  - each iteration is EVT (one event) then PASS (one head evaluation), so the pass that follows a tick's last
//    event runs in the same iteration;
//  - the tight fit compares against the level memories in the kernel's constant bank (no table loads);
//  - the four u64 accumulators stay in registers.
// ================================================================================================================
struct FFShared {
    uint32_t pinfo[16];                 // level | comp << 4 | lenmask << 8 (DevGeom::pinfo)
    uint32_t level_mem[8], level_next[8];
    uint32_t mem0, full_mem;
    uint8_t place_s[8][8];              // start slot of placement k of profile p
    uint8_t alloc[256 * 8];             // Alg. 2 by (occupancy, profile): start slot of the placement, 0xFF = FAIL
    uint32_t lmem[8];                   // level memories, padded with 0xFFFFFFFF (tight-fit binary search)
    uint8_t lvl_first[8];               // first profile of each level ([n_levels..] = 0xFF = none)
    uint8_t nobusy[256 * 8];            // placements of p touching no busy slot, by busy-slot mask
    unsigned long long reuse_sel[16];   // idle instances that tightly fit profile p (R7), over the IPM bytes
    uint16_t cbase[8];                  // fusion/fission-table column of candidate mask 0 of profile p
    unsigned long long key[8][kLaneThreads];  // per lane and start slot: end << 32 | (job | kind << 16) << 3 | slot
    uint32_t c32[kT32];
};

// Tight fit by a branch-free binary search over the 8 padded level memories in shared memory (3 loads).
#define FF_FIT_S(req)                                                  \
    ([&](uint32_t r_) {                                                \
        uint32_t L_ = S.lmem[3] < r_ ? 4u : 0u;                        \
        L_ += S.lmem[L_ + 1] < r_ ? 2u : 0u;                           \
        L_ += S.lmem[L_] < r_ ? 1u : 0u;                               \
        return (uint32_t)S.lvl_first[L_];                              \
    }(req))

__device__ __forceinline__ uint32_t ff_fit(const LaneParams& P, uint32_t req) {
    uint32_t L = 0;
#pragma unroll
    for (int l = 0; l < kMaxLevels; ++l) L += req > P.lm[l] ? 1u : 0u;
    const uint32_t p = (P.lfirst >> (4 * L)) & 0xFu;
    return p == 0xFu ? kNoNeed : p;
}

#ifndef FF_MINB
#define FF_MINB 8
#endif
// NS: the start slots scanned for the next event (every placement of the geometry starts below NS; A100: 7).
// KIND: MIG_FUSION_FISSION (Scheme B: idle instances persist and are reused, fused or split) or MIG_DYNAMIC (Alg. 2
// creates a tight slice on demand and the run's end destroys it, R10: no reuse, no fusion / fission).
// ORD: units are visited in P.order (trace_order.cu); the instantiations without it keep the plain unit counter.
template <int NS, bool XR, bool ER, int KIND, bool ORD>
__global__ void __launch_bounds__(kLaneThreads, FF_MINB) k_ff_lane(const DevGeom* __restrict__ Gg, const LaneParams P) {
    constexpr bool FF = KIND == MIG_FUSION_FISSION;
    __shared__ __align__(16) FFShared S;
    const uint32_t tid = threadIdx.x;
    {
        const DevGeom* G = Gg;
        for (uint32_t i = tid; i < 256 * 8; i += blockDim.x) {  // Alg. 2 for every (occupancy, profile)
            const uint32_t occ = i >> 3, p = i & 7u;
            const uint32_t np = __ldg(&G->n_prof), ns = __ldg(&G->n_slots);
            uint32_t best = 0, bk = 0xFFu, nb = 0;
            if (p < np) {
                const uint32_t npl = __ldg(&G->n_place[p]);
                for (uint32_t k = 0; k < npl; ++k) {
                    const uint32_t pl = __ldg(&G->place[p][k]), qm = pl >> 8;
                    if (occ < (1u << ns)) {
                        const uint32_t score =
                            (pl && !(occ & qm)) ? ((uint32_t)__ldg(&G->fcr[occ | qm]) << 8) | (pl & 0xFFu) : 0u;
                        if (score > best) {
                            best = score;
                            bk = pl & 0xFFu;  // the start slot of the best placement
                        }
                    }
                    nb |= (qm & occ) ? 0u : 1u << k;  // here occ plays the busy-slot mask
                }
            }
            S.alloc[i] = (uint8_t)bk;
            S.nobusy[i] = (uint8_t)nb;
        }
        if (tid < 16) {
            const uint32_t np = __ldg(&G->n_prof);
            uint32_t ok = 0;
            if (tid < np)
                for (uint32_t q = 0; q < np; ++q)
                    if (__ldg(&G->level[q]) == __ldg(&G->level[tid]) && __ldg(&G->comp[q]) >= __ldg(&G->comp[tid]))
                        ok |= 1u << q;
            unsigned long long sel = 0;
            for (uint32_t q = 0; q < 8; ++q)
                if ((ok >> q) & 1u) sel |= 0xFFull << (8 * q);
            S.reuse_sel[tid] = sel;
            S.pinfo[tid] = __ldg(&G->pinfo[tid]);
        }
        if (tid < 64) S.place_s[tid >> 3][tid & 7] = (uint8_t)__ldg(&G->place[tid >> 3][tid & 7]);
        if (tid < 8) {
            const uint32_t nl = __ldg(&G->n_levels), np = __ldg(&G->n_prof);
            S.level_mem[tid] = __ldg(&G->level_mem[tid]);
            S.level_next[tid] = __ldg(&G->level_next[tid]);
            S.lmem[tid] = tid < nl ? __ldg(&G->level_mem[tid]) : 0xFFFFFFFFu;
            uint32_t f = 0xFFu;
            for (uint32_t p = np; p-- > 0;)
                if (__ldg(&G->level[p]) == tid) f = p;
            S.lvl_first[tid] = (uint8_t)(tid < nl ? f : 0xFFu);
        }
        if (tid == 0) {
            uint32_t cb = 0;
            const uint32_t np = __ldg(&G->n_prof);
            for (uint32_t p = 0; p < 8; ++p) {
                S.cbase[p] = (uint16_t)cb;
                cb += p < np ? 1u << __ldg(&G->n_place[p]) : 0u;
            }
            S.mem0 = __ldg(&G->mem[0]);
            S.full_mem = __ldg(&G->full_mem);
        }
        if (tid < kT32) S.c32[tid] = 0;
#pragma unroll
        for (int f = 0; f < kT64; ++f) P.part[((size_t)blockIdx.x * kT64 + f) * kLaneThreads + tid] = 0;
    }
    __syncthreads();

    const uint32_t reconfig = P.pol.reconfig_ticks, ctx = P.ctx;
    const uint64_t jbase = P.off[0];
#define FF_RING (P.ring + (size_t)(blockIdx.x * kLaneThreads + tid) * P.ring_cap)
    unsigned long long* const key = &S.key[0][tid];
    constexpr unsigned long long kIdle = ~0ull;

    // A warp takes its units 32 at a time, and only once every lane has finished its trace: the lanes start their
    // traces together, so lanes holding alike traces (the visit order, ORD) step through them in phase. A lane that
    // finishes early waits (mode 4) for the others. (Config 2: FF launch 2.54 -> 2.04 ms; configs 3 / 4 / 5 k_simulate
    // 2.85 -> 2.54, 11.7 -> 8.4, 1652 -> 1555 ms against units taken one per lane as each finished.) Returns the
    // trace of this lane's unit, ~0 once the units are exhausted.
    const uint32_t lane = tid & 31u;
    auto take_batch = [&]() -> unsigned long long {
        unsigned long long u0 = 0;
        if (lane == 0) u0 = atomicAdd(P.counter, 32ull);
        u0 = __shfl_sync(FULL, u0, 0);
        return ORD ? lane_unit_trace(P, u0 + lane) : (u0 + lane < P.n_traces ? u0 + lane : ~0ull);
    };
    unsigned long long tr = take_batch();
    uint64_t j0 = 0;  // index of the unit's first job record
    uint32_t n = 0, err = 0, t = 0, qh = 0, rh = 0, rn = 0, mode = 0;
    uint32_t occ = 0, SM = 0, BS = 0, BM = 0, prof4 = 0;
    uint64_t IPM = 0;  // idle instances by profile: byte p bit s = an idle instance of profile p starts at s
    uint32_t K0 = 0, K1 = 0, K2 = 0, K3 = 0, hl = 0, hh = 0;
    unsigned long long a_turn = 0, a_busy = 0, a_mem = 0, a_waste = 0, kmin = kIdle;
    uint32_t hj = kNoJob, hneed = kUnk;
    uint4 hr = make_uint4(0, 0, 0, 0);

    auto fetch_head = [&]() {  // queue = jobs[qh..n) ++ requeue FIFO
        if (qh < n) {
            hj = qh;
            hneed = kUnk;
        } else if (rn) {
            const uint32_t v = FF_RING[rh];
            hj = v & 0x3FFu;
            hneed = v >> 10;
            if (hneed == 15u) hneed = kNoNeed;
        } else {
            hj = kNoJob;
            return;
        }
        hr = __ldg(P.jobs + j0 + hj);
        if (XR) {  // est + ws and true + ws (the context is added where they are used; true saturates, mig.h)
            const uint32_t ws = __ldg(&P.ext[j0 + hj].x);
            hr.x += ws;
            hr.y = hr.y + ws < hr.y ? 0xFFFFFFFFu : hr.y + ws;
        }
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
        t = qh = rh = rn = 0;
        occ = SM = BS = BM = prof4 = 0;
        IPM = 0;
#pragma unroll
        for (int k = 0; k < NS; ++k) key[k * kLaneThreads] = kIdle;
        kmin = kIdle;
        K0 = K1 = K2 = K3 = 0;
        a_turn = a_busy = a_mem = a_waste = 0;
        hl = (uint32_t)kFnvOffset;
        hh = (uint32_t)(kFnvOffset >> 32);
        mode = 0;
        fetch_head();
    };

    bool active = tr < P.n_traces;
    if (active) init_unit();
    else mode = 3;
    while (__any_sync(FULL, active)) {
        // ---- EVT: apply the event of kmin (R28 order), then refresh kmin ----
        if (mode == 1) {
            if (kmin == kIdle) {
                mode = 2;  // nothing running and nothing placeable: the unit is done
            } else {
                const uint32_t lo = (uint32_t)kmin, es = lo & 7u, job = (lo >> 3) & 0xFFFFu, ek = lo >> 19;
                t = (uint32_t)(kmin >> 32);
                const uint32_t epr = (prof4 >> (4 * es)) & 0xFu, si = S.pinfo[epr];
                const uint32_t elo = (job << 16) | (es << 8) | (epr << 4);
                lrec(hl, hh, t, elo | ((K_COMPLETE + ek) << 12));  // COMPLETE 6 / OOM 7 / PREEMPT 8
                if (ek == 0) {
                    a_turn += t;
                } else {  // OOM: next larger slice (R14) or FAILED on the whole GPU; PREEMPT (ER): the
                          // converged forecast, at most the whole GPU (R25)
                    uint32_t req;
                    if (ER && ek == 2) {
                        K3 += 1u;
                        req = min(__ldg(&P.est[j0 + job].pred_mib), S.full_mem);
                    } else {
                        K2 += 1u << 16;
                        req = S.level_next[si & 0xFu];
                    }
                    if (req == 0) {
                        lrec(hl, hh, t, elo | (K_FAILED << 12));
                        K3 += 1u << 16;
                    } else {  // back to the queue tail (R13) with the new tight fit
                        const uint32_t nn = ff_fit(P, req);
                        uint32_t pos = rh + rn;
                        if (pos >= P.ring_cap) pos -= P.ring_cap;
                        FF_RING[pos] = (uint16_t)(job | ((nn == kNoNeed ? 15u : nn) << 10));
                        ++rn;
                        if (hj == kNoJob) fetch_head();
                    }
                }
                key[es * kLaneThreads] = kIdle;
                const uint32_t ext = ((si >> 8) & 0xFFu) << es;
                BS &= ~(1u << es);
                BM &= ~ext;
                if (FF) {
                    IPM |= 1ull << (8 * epr + es);  // the instance is idle
                } else {  // DYNAMIC: freed at the run's end (R10)
                    occ &= ~ext;
                    K1 += 1u;
                }
                unsigned long long m = key[0];
#pragma unroll
                for (int k = 1; k < NS; ++k) m = min(m, key[k * kLaneThreads]);
                kmin = m;
                if ((uint32_t)(m >> 32) != t || m == kIdle) mode = 0;  // the tick is over: one scheduler pass
            }
        }
        __syncwarp();
        // ---- PASS: evaluate the head of the queue (Alg. 4, one decision) ----
        // P1 decides (kd, s, pr, nd) without branches on the common paths: the reuse candidates, the Alg. 2 answer and
        // the fusion/fission candidates are all looked up, then selected (REUSE before ALLOC before A7 before WAIT);
        // only the rare A7 table probe and the first evaluation of a job branch. The warp reconverges; P2 records,
        // creates, starts the run and pops, one copy for every decision kind.
        if (mode == 0 && hj == kNoJob) mode = 1;
        const bool pass = mode == 0;
        uint32_t kd = 0, s = 0, pr = 0, nd = 0;
        bool a7try = false;
        if (pass) {
            if (hneed == kUnk) {  // first evaluation of an initial queue entry: record checks + tight fit
                const uint32_t cls = (hr.z >> 16) & 0xFFu, T = hr.z & 0xFFFFu;
                if (cls > 2 || T > 4096) err |= (uint32_t)MIG_ERR_BAD_RECORD;
                hneed = FF_FIT_S(cls == kClassDynamic ? S.mem0 : hr.x + ctx);  // R16 / est + ctx (a2)
            }
            const uint32_t need = hneed;
            const bool rej = need == kNoNeed;  // no profile can ever hold the job: REJECT
            const uint32_t nq = rej ? 0u : need;
            const uint64_t x = FF ? IPM & S.reuse_sel[nq] : 0ull;  // idle slices that tightly fit (R7)
            uint32_t y = (uint32_t)x | (uint32_t)(x >> 32);
            y |= y >> 16;
            y |= y >> 8;
            const uint32_t cand = y & 0xFFu;
            const uint32_t a = S.alloc[(occ << 3) | nq];  // Alg. 2: its start, 0xFF = FAIL
            const uint32_t rsl = 31u - __clz(cand | 1u);
            pr = rej ? kNoNeed : cand ? (prof4 >> (4 * rsl)) & 0xFu : need;
            s = cand ? rsl : a;
            kd = rej ? K_REJECT : cand ? K_REUSE : a != 0xFFu ? K_ALLOC : K_WAIT;
            a7try = FF && kd == K_WAIT && (SM & ~BS);  // fusion / fission may place it (idle instances exist)
        }
        if (a7try) {  // A7 (R8): candidates touching no busy slot, the host-built answer table
            const uint32_t need = hneed;
            const uint32_t cm = S.nobusy[(BM << 3) | need];
            if (cm) {
                const uint32_t sid = __ldg(P.sid + (occ | (SM << 8)));
                const uint2 e = __ldg(P.a7 + (sid * P.n_a7 + S.cbase[need] + cm));
                if (e.x) {
                    s = e.x & 0xFFu;
                    nd = 15u - ((e.x >> 8) & 0xFFu);
                    const uint32_t rm = e.y & 0xFFu;
                    IPM &= ~(0x0101010101010101ull * (SM & rm));  // destroyed (idle) instances
                    occ &= ~rm;
                    SM &= ~rm;
                    kd = K_RECONF;
                }
            }
        }
        __syncwarp();
        if (pass) {
            const uint32_t j = hj;
            const bool place = kd <= K_RECONF, created = kd >= K_ALLOC && place;
            // the decision record: placements carry (slot, profile, #destroyed); WAIT / REJECT slot 0xF and the tight
            // fit (REJECT: 0xF)
            lrec(hl, hh, t, (j << 16) | (kd << 12) | (place ? (s << 8) | (pr << 4) | nd : 0xF00u | (pr << 4)));
            K0 += place ? (created ? 0x10001u : 1u) : 0u;
            K1 += kd == K_WAIT ? 1u << 16 : nd;
            K2 += kd == K_REJECT ? 1u : 0u;
            if (kd == K_WAIT) mode = 1;
            if (place) {
                // ---- create (ALLOC / RECONF, try_new_mig_slice PAPER.md:609) or take the idle slice, run start ----
                const uint32_t si = S.pinfo[pr];
                const uint32_t lm8 = (si >> 8) & 0xFFu;
                if (created) {
                    occ |= lm8 << s;
                    if (FF) SM |= 1u << s;
                    prof4 = (prof4 & ~(0xFu << (4 * s))) | (pr << (4 * s));
                } else if (FF) {
                    IPM &= ~(1ull << (8 * pr + s));
                }
                // start_run: end tick and kind (OOM > COMPLETE in one iteration, R29)
                const uint32_t rs = t + (created ? reconfig : 0u);
                const uint32_t lev = si & 0xFu, comp = (si >> 4) & 0xFu, T = hr.z & 0xFFFFu, ticks = hr.w;
                uint32_t dur, ek, it;
                if (((hr.z >> 16) & 0xFFu) != kClassDynamic) {
                    const uint32_t phys = hr.y + ctx < hr.y ? 0xFFFFFFFFu : hr.y + ctx;
                    ek = (T >= 1 && phys > S.level_mem[lev]) ? 1u : 0u;  // R12: static jobs OOM at iteration 1
                    it = ek ? 1u : T;
                    dur = it * ticks;
                    a_mem += (uint64_t)phys * dur;
                } else if (P.est) {
                    // every field the run needs is loaded up front (independent loads, one latency): the first
                    // exceed at this level, the memory integral up to it / to convergence / to the end
                    const mig_job_estimate* ej = P.est + j0 + j;
                    const uint32_t* ew = reinterpret_cast<const uint32_t*>(ej);
                    const uint32_t fe = __ldg(reinterpret_cast<const unsigned short*>(ej) + 6 + lev);
                    const uint32_t m_fe = __ldg(ew + 12 + lev), m_T = __ldg(ew + 18);
                    uint32_t m_run;
                    if (ER) {  // a10: preempt at the convergence iteration when the forecast exceeds this slice
                        const uint4 e0 = __ldg(reinterpret_cast<const uint4*>(ej));  // (req0, pred, conv | n, fe0 | fe1)
                        const uint2 pc = make_uint2(e0.x, e0.y);
                        const uint32_t conv = e0.z & 0xFFFFu;
                        const uint32_t m_conv = __ldg(ew + 17);
                        const uint32_t cap = S.level_mem[lev];
                        const uint32_t i_pre = (conv > 0 && pc.y > cap && cap < S.full_mem) ? conv : 0xFFFFFFFFu;
                        ek = fe <= min(T, i_pre) ? 1u : i_pre < T ? 2u : 0u;  // R29: OOM > COMPLETE > PREEMPT
                        it = ek == 1 ? fe : ek == 2 ? i_pre : T;
                        m_run = ek == 1 ? m_fe : ek == 2 ? m_conv : m_T;
                    } else {
                        ek = fe <= T ? 1u : 0u;
                        it = ek ? fe : T;
                        m_run = ek ? m_fe : m_T;
                    }
                    dur = it * ticks;
                    a_mem += (uint64_t)m_run * ticks;
                } else {  // a DYNAMIC record under MIG_TRACES_NO_DYNAMIC (no estimates): flagged, no forecast
                    err |= (uint32_t)MIG_ERR_BAD_RECORD;
                    ek = 0;
                    it = T;
                    dur = T * ticks;
                }
                if (((uint64_t)it * ticks + rs) >> 32) err |= (uint32_t)MIG_ERR_TICK_OVERFLOW;  // u32 ticks (mig.h)
                a_busy += (uint64_t)comp * dur;
                if (ek) a_waste += dur;
                const unsigned long long kk = ((unsigned long long)(rs + dur) << 32) | (((j | (ek << 16)) << 3) | s);
                key[s * kLaneThreads] = kk;
                kmin = min(kmin, kk);
                BS |= 1u << s;
                BM |= lm8 << s;
            }
            if (kd != K_WAIT) {  // pop the head
                if (qh < n) {
                    ++qh;
                } else {
                    rh = rh + 1 == P.ring_cap ? 0u : rh + 1u;
                    --rn;
                }
                fetch_head();
            }
        }
        __syncwarp();
        // ---- FIN: the unit's result (96 B) and totals; take the next unit ----
        if (mode == 2) {
            const uint32_t placements = K0 & 0xFFFFu, creates = K0 >> 16, destroys = K1 & 0xFFFFu, waits = K1 >> 16,
                           rejected = K2 & 0xFFFFu, ooms = K2 >> 16, preempts = K3 & 0xFFFFu, failed = K3 >> 16;
            const uint32_t completed = n - rejected - failed, restarts = ooms - failed + preempts;
            const uint32_t makespan = t;
            const uint64_t energy = (uint64_t)P.pol.idle_w * makespan + (uint64_t)P.pol.w_per_slice * a_busy;
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
            mode = 4;  // wait for the warp's other lanes
        }
        if (__all_sync(FULL, mode >= 3) && __any_sync(FULL, mode == 4)) {  // the warp's next 32 units
            tr = take_batch();
            if (tr < P.n_traces) {
                init_unit();
            } else {
                active = false;
                mode = 3;
            }
        }
    }
#undef FF_RING
    lane_flush_totals(P, S.c32);
}

// ================================================================================================================
// k_base_lane: the BASELINE launch of the common case (no extension records, no policy flags, no arrival streams).
// BASELINE is an in-order fold over the queue: each job waits for the previous one on the whole
// GPU, so a trace is one pass over its records with no event queue. One lane per trace; a warp takes 32 consecutive
// traces and advances them one job per iteration in lockstep (the record of job k+1 is loaded while job k is
// folded). Records, counters and results are those of k_simulate_lane<MIG_BASELINE> (same parity suites):
//   per job j, at tick t:  REJECT(j) if no profile holds it; else [WAIT(j) at t, the previous run's end at its end
//   tick (COMPLETE, or OOM + FAILED on the whole GPU), t = that tick] then PLACE_BASELINE(j) at t.
// ================================================================================================================
#ifndef BASE_MINB
#define BASE_MINB 8
#endif
template <bool XR>
__global__ void __launch_bounds__(kLaneThreads, BASE_MINB) k_base_lane(const DevGeom* __restrict__ Gg, const LaneParams P) {
    __shared__ uint32_t c32[kT32];
    const uint32_t tid = threadIdx.x, lane = tid & 31u;
    if (tid < kT32) c32[tid] = 0;
#pragma unroll
    for (int f = 0; f < kT64; ++f) P.part[((size_t)blockIdx.x * kT64 + f) * kLaneThreads + tid] = 0;
    const uint32_t fp = __ldg(&Gg->full_prof);
    const uint32_t fsi = __ldg(&Gg->pinfo[fp]);
    const uint32_t flev = fsi & 0xFu, fcomp = (fsi >> 4) & 0xFu, fcap = __ldg(&Gg->level_mem[flev]);
    const uint32_t mem0 = __ldg(&Gg->mem[0]);
    const uint32_t ctx = P.ctx;
    const uint64_t jbase = P.off[0];
    __syncthreads();
    unsigned long long p_make = 0, p_turn = 0, p_busy = 0, p_hash = 0, p_mem = 0, p_waste = 0;
    for (;;) {
        unsigned long long w0 = 0;
        if (lane == 0) w0 = atomicAdd(P.counter, 32ull);
        w0 = __shfl_sync(FULL, w0, 0);
        if (w0 >= P.n_traces) break;
        const unsigned long long tr = w0 + lane;
        const bool act = tr < P.n_traces;
        uint64_t j0 = 0;
        uint32_t n = 0, err = 0;
        if (act) {
            const uint64_t o0 = P.off[tr], o1 = P.off[tr + 1];
            j0 = o0 - jbase;
            n = (uint32_t)(o1 - o0);
            if (o1 - o0 > P.max_jobs) {
                err = (uint32_t)MIG_ERR_TRACE_TOO_LONG;
                n = 0;
            }
        }
        const uint32_t nmax = __reduce_max_sync(FULL, n);
        uint32_t t = 0, bend = 0, bjob = 0, hl = (uint32_t)kFnvOffset, hh = (uint32_t)(kFnvOffset >> 32);
        uint32_t placements = 0, waits = 0, rejected = 0, failed = 0;
        bool busy = false, boom = false;
        unsigned long long a_turn = 0, a_busy = 0, a_mem = 0, a_waste = 0;
        const uint4* rec = P.jobs + j0;
        const uint4* xrec = XR ? P.ext + j0 : nullptr;
        uint4 r = n ? __ldg(rec) : make_uint4(0, 0, 0, 0);
        uint32_t w = XR && n ? __ldg(&xrec[0].x) : 0u;  // the job's workspace MiB (extension record)
        for (uint32_t k = 0; k < nmax; ++k) {
            const uint4 rn = (k + 1 < n) ? __ldg(rec + k + 1) : make_uint4(0, 0, 0, 0);  // one ahead
            const uint32_t wn = XR && k + 1 < n ? __ldg(&xrec[k + 1].x) : 0u;
            if (XR) {  // est + ws, true + ws (saturating, as k_simulate_lane's 64-bit sum)
                r.x += w;
                r.y = r.y + w < r.y ? 0xFFFFFFFFu : r.y + w;
            }
            if (k < n) {
                const uint32_t cls = (r.z >> 16) & 0xFFu, T = r.z & 0xFFFFu, j = k;
                if (cls > 2 || T > 4096) err |= (uint32_t)MIG_ERR_BAD_RECORD;
                const uint32_t need = ff_fit(P, cls == kClassDynamic ? mem0 : r.x + ctx);  // R16 / est + ctx
                if (need == kNoNeed) {  // no profile can ever hold the job: REJECT (no wait)
                    lrec(hl, hh, t, (j << 16) | (K_REJECT << 12) | 0xFF0u);
                    ++rejected;
                } else {
                    if (busy) {  // the head waits for the running job, then its end event
                        lrec(hl, hh, t, (j << 16) | (K_WAIT << 12) | 0xF00u | (need << 4));
                        ++waits;
                        t = bend;
                        const uint32_t lo = (bjob << 16) | (fp << 4);
                        if (boom) {  // OOM on the whole GPU = FAILED
                            lrec(hl, hh, t, lo | (K_OOM << 12));
                            lrec(hl, hh, t, lo | (K_FAILED << 12));
                            ++failed;
                        } else {
                            lrec(hl, hh, t, lo | (K_COMPLETE << 12));
                            a_turn += t;
                        }
                    }
                    lrec(hl, hh, t, (j << 16) | (K_PLACE_BASELINE << 12) | (fp << 4));
                    ++placements;
                    // start_run on the whole GPU (OOM > COMPLETE in one iteration, R29)
                    const uint32_t ticks = r.w;
                    uint32_t dur, ek, it;
                    if (cls != kClassDynamic) {
                        const uint32_t phys = r.y + ctx < r.y ? 0xFFFFFFFFu : r.y + ctx;
                        ek = (T >= 1 && phys > fcap) ? 1u : 0u;  // R12: static jobs OOM at iteration 1
                        it = ek ? 1u : T;
                        dur = it * ticks;
                        a_mem += (uint64_t)phys * dur;
                    } else if (P.est) {  // independent loads: the first exceed and both memory integrals
                        const mig_job_estimate* ej = P.est + j0 + j;
                        const uint32_t* ew = reinterpret_cast<const uint32_t*>(ej);
                        const uint32_t fe = __ldg(reinterpret_cast<const unsigned short*>(ej) + 6 + flev);
                        const uint32_t m_fe = __ldg(ew + 12 + flev), m_T = __ldg(ew + 18);
                        ek = fe <= T ? 1u : 0u;
                        it = ek ? fe : T;
                        dur = it * ticks;
                        a_mem += (uint64_t)(ek ? m_fe : m_T) * ticks;
                    } else {  // DYNAMIC under MIG_TRACES_NO_DYNAMIC: flagged, no forecast
                        err |= (uint32_t)MIG_ERR_BAD_RECORD;
                        ek = 0;
                        it = T;
                        dur = T * ticks;
                    }
                    if (((uint64_t)it * ticks + t) >> 32) err |= (uint32_t)MIG_ERR_TICK_OVERFLOW;  // u32 ticks
                    a_busy += (uint64_t)fcomp * dur;
                    if (ek) a_waste += dur;
                    bend = t + dur;
                    bjob = j;
                    boom = ek != 0;
                    busy = true;
                }
            }
            r = rn;
            w = wn;
        }
        if (busy) {  // the last run's end
            t = bend;
            const uint32_t lo = (bjob << 16) | (fp << 4);
            if (boom) {
                lrec(hl, hh, t, lo | (K_OOM << 12));
                lrec(hl, hh, t, lo | (K_FAILED << 12));
                ++failed;
            } else {
                lrec(hl, hh, t, lo | (K_COMPLETE << 12));
                a_turn += t;
            }
        }
        if (act) {
            const uint32_t ooms = failed, completed = n - rejected - failed, makespan = t;
            const uint64_t energy = (uint64_t)P.pol.idle_w * makespan + (uint64_t)P.pol.w_per_slice * a_busy;
            if (P.out) {
                uint4* o = reinterpret_cast<uint4*>(P.out + tr * P.n_pol_all + P.pol_idx);
                o[0] = make_uint4(makespan, n, completed, rejected);
                o[1] = make_uint4(failed, ooms, 0u, ooms - failed);
                o[2] = make_uint4(placements, waits, 0u, 0u);
                o[3] = make_uint4((uint32_t)energy, (uint32_t)(energy >> 32), (uint32_t)a_turn,
                                  (uint32_t)(a_turn >> 32));
                o[4] = make_uint4((uint32_t)a_busy, (uint32_t)(a_busy >> 32), hl, hh);
                o[5] = make_uint4((uint32_t)a_mem, (uint32_t)(a_mem >> 32), (uint32_t)a_waste,
                                  (uint32_t)(a_waste >> 32));
            }
            atomicAdd(c32 + 0, 1u);
            atomicAdd(c32 + 1, n);
            if (rejected) atomicAdd(c32 + 2, rejected);
            if (failed) {
                atomicAdd(c32 + 3, failed);
                atomicAdd(c32 + 4, ooms);
            }
            atomicAdd(c32 + 6, placements);
            if (waits) atomicAdd(c32 + 7, waits);
            atomicMax(c32 + 10, makespan);
            if (err) atomicOr(c32 + 11, err);
            p_make += makespan;
            p_turn += a_turn;
            p_busy += a_busy;
            p_hash += ((unsigned long long)hh << 32) | hl;
            p_mem += a_mem;
            p_waste += a_waste;
        }
    }
    {
        unsigned long long* d = P.part + (size_t)blockIdx.x * kT64 * kLaneThreads + tid;
        d[0 * kLaneThreads] = p_make;
        d[1 * kLaneThreads] = p_turn;
        d[2 * kLaneThreads] = p_busy;
        d[3 * kLaneThreads] = p_hash;
        d[4 * kLaneThreads] = p_mem;
        d[5 * kLaneThreads] = p_waste;
    }
    lane_flush_totals(P, c32);
}


cudaError_t launch_ff_lane(const DevGeom* Gdev, const LaneParams& P, uint32_t ns, uint64_t max_blocks, int sm_count,
                           cudaStream_t stream) {
    static int per_sm = 0;
    if (!per_sm) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_ff_lane<8, true, true, MIG_FUSION_FISSION, false>,
                                                      kLaneThreads, 0);
        if (per_sm < 1) per_sm = 1;
    }
    const dim3 grid((unsigned)std::min<uint64_t>(max_blocks, lane_blocks(per_sm, P.n_traces, sm_count))),
        block(kLaneThreads);
    const bool xr = P.ext != nullptr, er = (P.pol.flags & MIG_EARLY_RESTART) != 0;
    const bool dyn = P.pol.kind == MIG_DYNAMIC;
    // the visit order is used by the plain-record instantiations (the long homogeneous queues it helps)
    const bool ord = P.order != nullptr && !xr;
#define FF_LAUNCH_K(NS_, K_)                                                                       \
    if (xr && er) k_ff_lane<NS_, true, true, K_, false><<<grid, block, 0, stream>>>(Gdev, P);      \
    else if (xr) k_ff_lane<NS_, true, false, K_, false><<<grid, block, 0, stream>>>(Gdev, P);      \
    else if (er && ord) k_ff_lane<NS_, false, true, K_, true><<<grid, block, 0, stream>>>(Gdev, P); \
    else if (er) k_ff_lane<NS_, false, true, K_, false><<<grid, block, 0, stream>>>(Gdev, P);      \
    else if (ord) k_ff_lane<NS_, false, false, K_, true><<<grid, block, 0, stream>>>(Gdev, P);     \
    else k_ff_lane<NS_, false, false, K_, false><<<grid, block, 0, stream>>>(Gdev, P);
#define FF_LAUNCH(NS_)                           \
    if (dyn) {                                   \
        FF_LAUNCH_K(NS_, MIG_DYNAMIC)            \
    } else {                                     \
        FF_LAUNCH_K(NS_, MIG_FUSION_FISSION)     \
    }
    if (ns <= 4) {
        FF_LAUNCH(4)
    } else if (ns <= 7) {
        FF_LAUNCH(7)
    } else {
        FF_LAUNCH(8)
    }
#undef FF_LAUNCH
#undef FF_LAUNCH_K
    return cudaGetLastError();
}

cudaError_t launch_base_lane(const DevGeom* Gdev, const LaneParams& P, uint64_t max_blocks, int sm_count,
                             cudaStream_t stream) {
    static int per_sm = 0;
    if (!per_sm) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_base_lane<true>, kLaneThreads, 0);
        if (per_sm < 1) per_sm = 1;
    }
    const dim3 grid((unsigned)std::min<uint64_t>(max_blocks, lane_blocks(per_sm, P.n_traces, sm_count)));
    if (P.ext) k_base_lane<true><<<grid, kLaneThreads, 0, stream>>>(Gdev, P);
    else k_base_lane<false><<<grid, kLaneThreads, 0, stream>>>(Gdev, P);
    return cudaGetLastError();
}

}  // namespace mig
