// simulate.cu — k_simulate: the MIGM scheduler + partition-manager event loop over many independent traces
// (SURVEY.md §8(a) rows a1, a4-a12).
//
// One warp per trace (persistent CTAs, atomic trace counter). The trace's jobs are staged into shared memory
// (coalesced 128-bit loads, 32 B per job: iterations, class, tight-fit profile, iteration ticks, first
// requirement, warps, forecast, convergence iteration and the first-exceed iteration of every memory level).
// The partition state is lane-resident: lane s owns the instance that starts at memory slot s (profile, busy,
// job, end tick, end kind), and the occupancy is a warp-uniform bitmask. Every decision is lane-parallel:
//   tight fit / reuse / static choice ....... __ballot_sync over profiles or instances, __ffs / __clz
//   Alg. 2 ............... lane k scores placement k as (fcr[occ|mask] << 8 | start) from the
//                                             shared-memory fcr table and __reduce_max_sync picks the winner
//   fusion / fission ......... lane k scores (fcr[occ'] << 16 | (15 - #destroyed) << 8 | start)
//   next event ............................... __reduce_min_sync over the busy instances' end ticks, ties by
//                                             (kind, job) with a second __reduce_min_sync
// Counters are lane-distributed (lane c holds counter c); the per-trace decision stream is folded into an
// FNV-1a-64 hash. Per-trace results (80 B) are written with 128-bit stores and per-policy totals are reduced in
// shared memory then added to global memory once per CTA.
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
    mig_policy pol[kMaxPolicies];
};

// counters held by lane c
enum : uint32_t {
    C_COMPLETED = 0, C_REJECTED, C_FAILED, C_OOMS, C_PREEMPTS, C_RESTARTS, C_PLACEMENTS, C_WAITS, C_CREATES,
    C_DESTROYS, C_TURNAROUND, C_BUSY
};
#define CBIT(c) (1u << (c))

// Shared-memory image of the geometry (copied from the device-resident DevGeom once per CTA; lane-divergent
// table reads such as fcr[occ | mask] then hit shared memory instead of serialising on the constant bank).
constexpr size_t kGeomBytes = (sizeof(DevGeom) + 15) & ~size_t(15);
constexpr size_t kPolBytes = (kMaxPolicies * sizeof(mig_policy) + 15) & ~size_t(15);
constexpr size_t kTotBytes = kMaxPolicies * 20 * 8;

constexpr int kWarps = 8;  // warps (traces in flight) per CTA

__device__ __forceinline__ void bump(uint64_t& cnt, uint32_t lane, uint32_t mask, uint64_t v) {
    if ((mask >> lane) & 1u) cnt += v;
}

// Tight fit (R6, R30), lanes over profiles.
__device__ __forceinline__ uint32_t tight_fit_warp(const DevGeom& G, uint32_t req, uint32_t warps, bool fold,
                                                   uint32_t lane) {
    bool ok = lane < G.n_prof && G.mem[lane] >= req;
    if (fold && warps > 0 && lane < G.n_prof) {
        uint32_t cf = G.wave_cap[G.full_prof], cp = G.wave_cap[lane];
        ok = ok && ((warps + cp - 1) / cp == (warps + cf - 1) / cf);
    }
    uint32_t m = __ballot_sync(FULL, ok);
    return m ? (uint32_t)(__ffs(m) - 1) : 0xFFu;
}

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

__global__ void __launch_bounds__(kWarps * 32) k_simulate(const DevGeom* __restrict__ Gg, const SimParams P) {
    extern __shared__ __align__(16) uint8_t smem[];
    DevGeom& G = *reinterpret_cast<DevGeom*>(smem);
    mig_policy* s_pol = reinterpret_cast<mig_policy*>(smem + kGeomBytes);
    unsigned long long* s_tot = reinterpret_cast<unsigned long long*>(smem + kGeomBytes + kPolBytes);
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    const uint32_t per_warp = P.max_jobs * 32u + ((P.max_jobs * 2u + 15u) & ~15u) + 96u;
    uint8_t* wb = smem + kGeomBytes + kPolBytes + kTotBytes + warp * per_warp;
    uint4* jobA = reinterpret_cast<uint4*>(wb);                      // {T | cls<<16 | need<<24, ticks, req0, warps}
    uint4* jobB = jobA + P.max_jobs;                                 // {pred, conv | fe0<<16, fe1|fe2<<16, fe3|fe4<<16}
    uint16_t* ring = reinterpret_cast<uint16_t*>(jobB + P.max_jobs);  // requeue FIFO (R13: tail)
    uint32_t* sres = reinterpret_cast<uint32_t*>(wb + per_warp - 96u);  // 80 B result staging

    {
        const uint32_t* src = reinterpret_cast<const uint32_t*>(Gg);
        uint32_t* dst = reinterpret_cast<uint32_t*>(smem);
        for (uint32_t i = threadIdx.x; i < sizeof(DevGeom) / 4; i += blockDim.x) dst[i] = __ldg(src + i);
        if (threadIdx.x == 0) {
#pragma unroll
            for (int k = 0; k < kMaxPolicies; ++k) s_pol[k] = P.pol[k];
        }
        for (uint32_t i = threadIdx.x; i < kMaxPolicies * 20; i += blockDim.x) s_tot[i] = 0;
    }
    __syncthreads();
    const uint32_t full_mem = G.full_mem;

    const uint64_t j_base = P.off[0];
    for (;;) {
        unsigned long long tr = 0;
        if (lane == 0) tr = atomicAdd(P.counter, 1ull);
        tr = __shfl_sync(FULL, tr, 0);
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
        for (uint32_t j = lane; j < n; j += 32) {
            uint4 r = __ldg(P.jobs + j0 + j);
            uint4 e = P.ext ? __ldg(P.ext + j0 + j) : make_uint4(0, 0, 0, 0);
            const uint32_t cls = (r.z >> 16) & 0xFFu, T = r.z & 0xFFFFu;
            if (cls > 2 || T > 4096 || (r.z >> 24) != 0) err |= (uint32_t)MIG_ERR_BAD_RECORD;
            uint4 A, Bv;
            A.x = T | (cls << 16);
            A.y = r.w;
            A.w = e.y;
            if (cls == kClassDynamic) {
                const uint4* es = reinterpret_cast<const uint4*>(P.est + j0 + j);
                uint4 e0 = __ldg(es), e1 = __ldg(es + 1);
                A.z = e0.x;                                        // req0 (smallest slice, R16)
                Bv = make_uint4(e0.y, (e0.z & 0xFFFFu) | (e0.w << 16), (e0.w >> 16) | (e1.x << 16),
                                (e1.x >> 16) | (e1.y << 16));
            } else {
                A.z = r.x + e.x + P.ctx;                           // est + ws + ctx
                const uint64_t phys = (uint64_t)r.y + e.x + P.ctx;
                uint32_t fe[5];
#pragma unroll
                for (int l = 0; l < kMaxLevels; ++l)
                    fe[l] = (l < (int)G.n_levels && T >= 1 && phys > G.level_mem[l]) ? 1u : kNever;
                Bv = make_uint4(0u, fe[0] << 16, fe[1] | (fe[2] << 16), fe[3] | (fe[4] << 16));
            }
            jobA[j] = A;
            jobB[j] = Bv;
        }
        err = __reduce_or_sync(FULL, err);

        for (uint32_t p = 0; p < P.n_pol; ++p) {
            const mig_policy& pol = s_pol[p];
            const uint32_t kind = pol.kind;
            const bool fold = (pol.flags & MIG_WARP_FOLD) != 0;
            const bool er = (pol.flags & MIG_EARLY_RESTART) != 0 && kind != MIG_BASELINE;
            __syncwarp();
            for (uint32_t j = lane; j < n; j += 32) {
                uint4 A = jobA[j];
                A.x = (A.x & 0x00FFFFFFu) | (tight_fit_lane(G, A.z, A.w, fold) << 24);
                jobA[j].x = A.x;
            }
            __syncwarp();
            // ---- lane-resident instance table (lane s = instance starting at slot s) ----
            int ip = -1;  // profile
            uint32_t ibusy = 0, ijob = 0, iend = 0, ikind = 0;
            uint32_t occ = 0;
            if (kind == MIG_BASELINE) {
                if (lane == 0) ip = (int)G.full_prof;
                occ = G.lenmask[G.full_prof];
            } else if (kind == MIG_STATIC) {
                for (uint32_t i = 0; i < G.n_layout; ++i) {
                    if (lane == G.layout_start[i]) ip = (int)G.layout_prof[i];
                    occ |= G.lenmask[G.layout_prof[i]] << G.layout_start[i];
                }
            }
            uint64_t cnt = 0;  // lane-distributed counters
            uint64_t hash = kFnvOffset;
            uint32_t t = 0, makespan = 0;
            uint32_t qh = 0, rh = 0, rn = 0;  // queue = jobs[qh..n) ++ ring[rh .. rh+rn)

            // ---- a8: scheduler pass (Alg. 4; head-of-line, wake on every event R9) ----
            auto sched_pass = [&]() {
                while (qh < n || rn != 0) {
                    const uint32_t j = qh < n ? qh : (uint32_t)ring[rh];
                    const uint4 A = jobA[j];
                    const uint32_t need = A.x >> 24;
                    uint32_t s = 0xFFu, prof = 0, kd = 0, nd = 0;
                    bool created = false;
                    if (need == 0xFFu) {  // no profile can ever hold the job
                        hash_record(hash, t, j, K_REJECT, 0xF, 0xF, 0);
                        bump(cnt, lane, CBIT(C_REJECTED), 1);
                    } else {
                        const uint32_t nmem = G.mem[need], ncomp = G.comp[need];
                        if (kind == MIG_BASELINE || kind == MIG_STATIC) {
                            // smallest idle fitting slice, tie -> highest start (R11); baseline = whole GPU
                            const bool cand = ip >= 0 && G.mem[ip] >= nmem && G.comp[ip] >= ncomp;
                            const uint32_t key = (cand && !ibusy) ? (((31u - G.level[ip]) << 5) | lane) + 1u : 0u;
                            const uint32_t km = __reduce_max_sync(FULL, key);
                            if (km) {
                                s = (km - 1u) & 31u;
                                prof = (uint32_t)__shfl_sync(FULL, ip, s);
                                kd = kind == MIG_BASELINE ? K_PLACE_BASELINE : K_PLACE_STATIC;
                            } else if (__ballot_sync(FULL, cand)) {
                                kd = K_WAIT;
                            } else {
                                kd = K_REJECT;
                            }
                        } else {
                            if (kind == MIG_FUSION_FISSION) {  // idle slice that tightly fits (R7)
                                const bool cand = ip >= 0 && !ibusy && G.mem[ip] == nmem && G.comp[ip] >= ncomp;
                                const uint32_t m = __ballot_sync(FULL, cand);
                                if (m) {
                                    s = 31u - __clz(m);
                                    prof = (uint32_t)__shfl_sync(FULL, ip, s);
                                    kd = K_REUSE;
                                }
                            }
                            if (!kd) {  // Alg. 2: argmax fcr over legal placements, tie -> highest start (R5)
                                const uint32_t np = G.n_place[need];
                                uint32_t score = 0;
                                if (lane < np) {
                                    const uint32_t pl = G.place[need][lane], mask = pl >> 8;
                                    if (!(occ & mask)) score = ((uint32_t)G.fcr[occ | mask] << 8) | (pl & 0xFFu);
                                }
                                const uint32_t best = __reduce_max_sync(FULL, score);
                                if (best) {
                                    s = best & 0xFFu;
                                    prof = need;
                                    kd = K_ALLOC;
                                    created = true;
                                    occ |= G.lenmask[need] << s;
                                    if (lane == s) ip = (int)need;
                                } else if (kind == MIG_FUSION_FISSION) {
                                    // fusion/fission (R8): destroy the idle instances a
                                    // placement overlaps, best (fcr(result), -#destroyed, start)
                                    const uint32_t ext_l = ip >= 0 ? G.lenmask[ip] << lane : 0u;
                                    const uint32_t busy_slots = __reduce_or_sync(FULL, ibusy ? ext_l : 0u);
                                    uint32_t qm = 0, qs = 0;
                                    bool cand = false;
                                    if (lane < np) {
                                        const uint32_t pl = G.place[need][lane];
                                        qm = pl >> 8;
                                        qs = pl & 0xFFu;
                                        cand = !(qm & busy_slots) && (qm & occ);
                                    }
                                    uint32_t removed = 0, ndl = 0;
                                    for (uint32_t k = 0; k < G.n_slots; ++k) {
                                        const uint32_t ek = __shfl_sync(FULL, ext_l, k);
                                        if (ek & qm) {
                                            removed |= ek;
                                            ++ndl;
                                        }
                                    }
                                    const uint32_t sc =
                                        cand ? (((uint32_t)G.fcr[(occ & ~removed) | qm] << 16) | ((15u - ndl) << 8) | qs)
                                             : 0u;
                                    const uint32_t bs = __reduce_max_sync(FULL, sc);
                                    if (bs) {
                                        s = bs & 0xFFu;
                                        nd = 15u - ((bs >> 8) & 0xFFu);
                                        const uint32_t qmask = G.lenmask[need] << s;
                                        const bool kill = (ext_l & qmask) != 0;
                                        const uint32_t rem = __reduce_or_sync(FULL, kill ? ext_l : 0u);
                                        if (kill) ip = -1;
                                        occ = (occ & ~rem) | qmask;
                                        if (lane == s) ip = (int)need;
                                        prof = need;
                                        kd = K_RECONF;
                                        created = true;
                                    }
                                }
                                if (!kd) kd = K_WAIT;
                            }
                        }
                        if (kd == K_WAIT) {
                            hash_record(hash, t, j, K_WAIT, 0xF, need, 0);
                            bump(cnt, lane, CBIT(C_WAITS), 1);
                            return;  // head-of-line: the pass ends
                        }
                        if (kd == K_REJECT) {
                            hash_record(hash, t, j, K_REJECT, 0xF, need, 0);
                            bump(cnt, lane, CBIT(C_REJECTED), 1);
                        } else {
                            hash_record(hash, t, j, kd, s, prof, nd);
                            bump(cnt, lane, CBIT(C_PLACEMENTS) | (created ? CBIT(C_CREATES) : 0u), 1);
                            bump(cnt, lane, CBIT(C_DESTROYS), nd);
                            // ---- start the run; OOM / early restart / completion ----
                            const uint4 Bv = jobB[j];
                            const uint32_t T = A.x & 0xFFFFu, cls = (A.x >> 16) & 0xFFu, ticks = A.y;
                            const uint32_t cap = G.mem[prof];
                            const uint32_t fe = reinterpret_cast<const uint16_t*>(&jobB[j])[3 + G.level[prof]];
                            const uint32_t rs = t + (created ? pol.reconfig_ticks : 0u);
                            uint32_t i_pre = 0xFFFFFFFFu;
                            const uint32_t conv = Bv.y & 0xFFFFu;
                            if (er && cls == kClassDynamic && conv > 0 && Bv.x > cap && cap < full_mem) i_pre = conv;
                            uint32_t end, ek;
                            if (fe != kNever && fe <= min(T, i_pre)) {  // OOM > COMPLETE > PREEMPT (R29)
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
                                ibusy = 1;
                                ijob = j;
                                iend = end;
                                ikind = ek;
                            }
                            bump(cnt, lane, CBIT(C_BUSY), (uint64_t)G.comp[prof] * (end - rs));
                        }
                    }
                    // pop the head
                    if (qh < n) {
                        ++qh;
                    } else {
                        rh = rh + 1 == P.ring_cap ? 0 : rh + 1;
                        --rn;
                    }
                }
            };

            sched_pass();
            // ---- a8-a10: event loop ----
            for (;;) {
                const uint32_t mine = (ip >= 0 && ibusy) ? iend : 0xFFFFFFFFu;
                const uint32_t tn = __reduce_min_sync(FULL, mine);
                if (tn == 0xFFFFFFFFu) break;
                t = tn;
                uint32_t evm = __ballot_sync(FULL, mine == t);
                while (evm) {
                    uint32_t s;
                    if ((evm & (evm - 1u)) == 0u) {
                        s = (uint32_t)__ffs(evm) - 1u;
                    } else {  // several events at one tick: COMPLETE < OOM < PREEMPT, then job id (R28)
                        const uint32_t key = ((evm >> lane) & 1u) ? ((ikind << 16) | ijob) : 0xFFFFFFFFu;
                        const uint32_t km = __reduce_min_sync(FULL, key);
                        s = (uint32_t)__ffs(__ballot_sync(FULL, key == km)) - 1u;
                    }
                    evm &= ~(1u << s);
                    const uint32_t prof = (uint32_t)__shfl_sync(FULL, ip, s);
                    const uint32_t job = __shfl_sync(FULL, ijob, s);
                    const uint32_t ek = __shfl_sync(FULL, ikind, s);
                    bool requeue = false;
                    uint32_t req = 0;
                    if (ek == 0) {
                        hash_record(hash, t, job, K_COMPLETE, s, prof, 0);
                        bump(cnt, lane, CBIT(C_COMPLETED), 1);
                        bump(cnt, lane, CBIT(C_TURNAROUND), t);
                    } else if (ek == 1) {  // OOM: next larger slice (R14) or FAILED at full GPU
                        hash_record(hash, t, job, K_OOM, s, prof, 0);
                        const uint32_t nl = G.level_next[G.level[prof]];
                        if (nl == 0) {
                            hash_record(hash, t, job, K_FAILED, s, prof, 0);
                            bump(cnt, lane, CBIT(C_OOMS) | CBIT(C_FAILED), 1);
                        } else {
                            bump(cnt, lane, CBIT(C_OOMS) | CBIT(C_RESTARTS), 1);
                            requeue = true;
                            req = nl;
                        }
                    } else {  // PREEMPT: restart on the slice meeting the forecast (R25)
                        hash_record(hash, t, job, K_PREEMPT, s, prof, 0);
                        bump(cnt, lane, CBIT(C_PREEMPTS) | CBIT(C_RESTARTS), 1);
                        requeue = true;
                        req = min(jobB[job].x, full_mem);
                    }
                    if (requeue) {  // back to the queue tail (R13) with the new tight fit
                        const uint32_t need = tight_fit_warp(G, req, jobA[job].w, fold, lane);
                        __syncwarp();
                        if (lane == 0) {
                            jobA[job].x = (jobA[job].x & 0x00FFFFFFu) | (need << 24);
                            uint32_t pos = rh + rn;
                            if (pos >= P.ring_cap) pos -= P.ring_cap;
                            ring[pos] = (uint16_t)job;
                        }
                        __syncwarp();
                        ++rn;
                    }
                    if (lane == s) ibusy = 0;
                    if (kind == MIG_DYNAMIC) {  // free on completion (R10)
                        if (lane == s) ip = -1;
                        occ &= ~(G.lenmask[prof] << s);
                        bump(cnt, lane, CBIT(C_DESTROYS), 1);
                    }
                }
                makespan = t;
                sched_pass();
            }
            // ---- a11: per-trace result (80 B) ----
            const uint64_t busy = __shfl_sync(FULL, cnt, C_BUSY);
            __syncwarp();
            if (lane < 10) sres[2 + lane] = (uint32_t)cnt;
            if (lane == 0) {
                sres[0] = makespan;
                sres[1] = n;
            }
            uint64_t* sres64 = reinterpret_cast<uint64_t*>(sres);
            if (lane == C_TURNAROUND) sres64[7] = cnt;
            if (lane == C_BUSY) {
                sres64[8] = cnt;
                sres64[6] = (uint64_t)pol.idle_w * makespan + (uint64_t)pol.w_per_slice * busy;
            }
            if (lane == 12) sres64[9] = hash;
            __syncwarp();
            if (P.out && lane < 5)
                reinterpret_cast<uint4*>(P.out + tr * P.n_pol + p)[lane] = reinterpret_cast<const uint4*>(sres)[lane];
            // ---- a12: per-policy totals (shared-memory atomics, flushed once per CTA) ----
            if (lane < 19) {
                uint64_t v;
                if (lane == 0) v = 1;
                else if (lane < 12) v = sres[lane];
                else if (lane == 12 || lane == 13) v = sres[0];
                else if (lane == 18) v = err;
                else v = sres64[lane - 8];  // 14 energy, 15 turnaround, 16 busy, 17 hash
                if (lane == 13) atomicMax(&s_tot[p * 20 + 13], (unsigned long long)v);
                else if (lane == 18) { if (v) atomicOr(&s_tot[p * 20 + 18], (unsigned long long)v); }
                else atomicAdd(&s_tot[p * 20 + lane], (unsigned long long)v);
            }
        }
    }
    __syncthreads();
    if (P.totals && blockIdx.x == 0 && threadIdx.x < P.n_pol && P.est_err && *P.est_err)
        atomicOr(reinterpret_cast<unsigned long long*>(P.totals + threadIdx.x) + 18, *P.est_err);
    if (P.totals) {
        for (uint32_t i = threadIdx.x; i < P.n_pol * 20; i += blockDim.x) {
            unsigned long long* dst = reinterpret_cast<unsigned long long*>(P.totals) + i;
            const uint32_t f = i % 20;
            if (f == 13) atomicMax(dst, s_tot[i]);
            else if (f == 18) { if (s_tot[i]) atomicOr(dst, s_tot[i]); }
            else if (f < 18) atomicAdd(dst, s_tot[i]);
        }
    }
}

size_t simulate_smem_bytes(uint32_t max_jobs) {
    const size_t per_warp = (size_t)max_jobs * 32u + ((max_jobs * 2u + 15u) & ~15u) + 96u;
    return kGeomBytes + kPolBytes + kTotBytes + kWarps * per_warp;
}

cudaError_t launch_simulate(const DevGeom* Gdev, const mig_traces& tr, const mig_policy* pols, uint32_t n_pol,
                            const mig_job_estimate* est, mig_trace_result* out, mig_policy_totals* totals,
                            unsigned long long* counter, const unsigned long long* est_err, int sm_count,
                            cudaStream_t stream) {
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
    P.n_pol = n_pol;
    P.ctx = pols[0].ctx_mib;
    for (uint32_t i = 0; i < n_pol; ++i) P.pol[i] = pols[i];
    const size_t smem = simulate_smem_bytes(tr.max_jobs);
    cudaError_t e = cudaFuncSetAttribute(k_simulate, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_simulate, kWarps * 32, smem);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    uint64_t want = (tr.n_traces + kWarps - 1) / kWarps;
    uint64_t blocks = (uint64_t)per_sm * sm_count;
    if (want < blocks) blocks = want;
    if (blocks < 1) blocks = 1;
    k_simulate<<<(unsigned)blocks, kWarps * 32, smem, stream>>>(Gdev, P);
    return cudaGetLastError();
}

}  // namespace mig
