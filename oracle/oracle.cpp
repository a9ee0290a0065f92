// oracle.cpp — CPU ORACLE. TEST INFRASTRUCTURE ONLY.
//
// A plain, slow, obviously-correct, single-threaded C++ discrete-event simulator of the MIGM method
// (arXiv 2508.18556). Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
// load or execute it. It shares no code with the CUDA path (paper_2508_18556_b200/csrc); the only common code is the
// seeded INPUT generator tracegen/tracegen.h, used here to draw the per-iteration memory samples a dynamic job
// reports.
//
// Every function cites the passage it follows. Readings of silent/ambiguous passages are the R-numbers of
// DESIGN.md §"Readings" (= SURVEY.md §8(c) ambiguity register). Structure:
//   Geometry ........ §4.1 profiles + placement table (R1)
//   Alg. 1 .......... precompute_reachability: enumerate valid states S literally as sets of
//                     placed instances, finals F = states with no legal allocation (R2), fcr(s) = |reachable F| (R3)
//   Alg. 2 .......... allocate_partition: enumerate placements C, FAIL if empty, argmax fcr,
//                     tie -> highest start (R5)
//   Alg. 3 .......... PeakMemoryPrediction: per-iteration append, OLS fits of requested memory
//                     and inverse reuse ratio, forecast at max_iter with z*sigma, convergence (R18-R24, R37)
//   Alg. 4 .......... schedule_dyn_reconfig, Scheme B + fusion/fission (R8),
//                     OOM restart (R12-R15), early restart (R25),
//                     baseline, static slices (R11), dynamic (create/free)
//   Metrics ......... makespan, completions, energy (R26), turnaround, decision hash
//   or_reach ........ Alg. 1 for an arbitrary slot geometry given by placement masks (up to 20 slots), by the same
//                     literal definition (R42), the reference of mig_reachability
//
// Parity status of each function: see DESIGN.md §"Oracle pins". Nothing here is "parity unpinned": the EWMA variant
// (R36), which the paper does not describe, is pinned by hand-worked level sequences.

#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <functional>
#include <cmath>
#include <deque>
#include <map>
#include <queue>
#include <string>
#include <vector>

#include "../tracegen/tracegen.h"

namespace {

constexpr uint16_t NEVER = 0xFFFF;

// ---------------------------------------------------------------------------------------------------------------
// Plain C layouts exchanged with the Python test harness (oracle/oracle.py). Oracle-owned definitions.
// ---------------------------------------------------------------------------------------------------------------
struct OrGeomDesc {
    uint32_t n_slots, slot_mib, n_compute, sms_per_slice, warps_per_sm;
    uint32_t n_prof;
    uint32_t prof_compute[16], prof_len[16], prof_nstart[16], prof_start[16][8];
    uint32_t n_layout;
    uint32_t layout_prof[8], layout_start[8];
    uint32_t n_alay[8];                      // Scheme A homogeneous layout per memory level (R38)
    uint32_t alay_prof[8][8], alay_start[8][8];
};

struct OrPolicy {
    uint32_t kind;   // 0 BASELINE, 1 STATIC, 2 DYNAMIC, 3 FUSION_FISSION, 4 SCHEME_A
    uint32_t flags;  // 1 EARLY_RESTART, 2 WARP_FOLD, 4 EWMA_REUSE, 8 WAVE_TIME, 16 PCIE_CONTENTION
    uint32_t ctx_mib, reconfig_ticks, idle_w, w_per_slice;
    double z;
    uint32_t eps_num, eps_den, conv_k, min_n;
};

struct OrEstimate {  // 80 B
    uint32_t req0_mib, pred_mib;
    uint16_t conv_iter, n_levels;
    uint16_t fe[6];
    double phi, a, sigma;
    uint32_t mem_fe[5], mem_conv, mem_T, pad;  // sum of physical MiB over iterations 1..k, k = fe[l], conv, T
};

struct OrResult {  // 80 B
    uint32_t makespan, n_jobs, completed, rejected, failed, ooms, preempts, restarts, placements, waits, creates,
        destroys;
    uint64_t energy_wticks, turnaround_sum, busy_slice_ticks, decision_hash;
    uint64_t mem_mib_ticks;  // integral of the running jobs' physical memory over time
    uint64_t wasted_ticks;   // time of runs that ended in OOM or early restart
};
static_assert(sizeof(OrEstimate) == 80, "estimate layout");
static_assert(sizeof(OrResult) == 96, "result layout");

enum { BASELINE = 0, STATIC = 1, DYNAMIC = 2, FUSION_FISSION = 3, SCHEME_A = 4 };
enum { F_EARLY_RESTART = 1, F_WARP_FOLD = 2, F_EWMA = 4, F_WAVE_TIME = 8, F_PCIE = 16 };
enum { K_REUSE = 1, K_ALLOC, K_RECONF, K_WAIT, K_REJECT, K_COMPLETE, K_OOM, K_PREEMPT, K_FAILED, K_PLACE_STATIC,
       K_PLACE_BASELINE, K_LAYOUT, K_PLACE_GROUP };

// ---------------------------------------------------------------------------------------------------------------
// Geometry and Algorithm 1.
// ---------------------------------------------------------------------------------------------------------------
struct Placement {
    int prof, start, len;
};

struct Geometry {
    OrGeomDesc d;
    std::vector<Placement> pl;                 // every legal (profile, start) pair (R1)
    std::map<std::vector<int>, int> index;     // canonical state key (sorted placement ids) -> state id
    std::vector<std::vector<int>> states;      // S
    std::vector<std::vector<int>> succ;        // alloc edges delta(s, alloc(x))
    std::vector<int> final_id;                 // -1 or index into F
    std::vector<uint32_t> fcr;                 // fcr(s) = |F_s|
    uint32_t n_finals = 0;

    uint32_t mem(int p) const { return d.prof_len[p] * d.slot_mib; }
    uint32_t full_mem() const { return d.n_slots * d.slot_mib; }
    int placement_id(int prof, int start) const {
        for (size_t i = 0; i < pl.size(); ++i)
            if (pl[i].prof == prof && pl[i].start == start) return (int)i;
        return -1;
    }
};

bool overlaps(const Placement& a, const Placement& b) {
    return a.start < b.start + b.len && b.start < a.start + a.len;
}

// A placement may be added to a state iff it overlaps no placed instance and the compute
// slices stay within the GPU.
bool can_add(const Geometry& g, const std::vector<int>& s, int q) {
    uint32_t comp = g.d.prof_compute[g.pl[q].prof];
    for (int i : s) {
        if (i == q || overlaps(g.pl[i], g.pl[q])) return false;
        comp += g.d.prof_compute[g.pl[i].prof];
    }
    return comp <= g.d.n_compute;
}

std::vector<int> with(std::vector<int> s, int q) {
    s.push_back(q);
    std::sort(s.begin(), s.end());
    return s;
}

// "Enumerate all valid partition states S": breadth-first from s0 = unpartitioned GPU
// over single allocations; finals = states with no legal allocation (R2); then
// "for each valid partition state s: compute all reachable fully configured states F_s; fcr(s) <- |F_s|"
// by a memoised depth-first union over the alloc edges.
std::string build_geometry(Geometry& g) {
    const OrGeomDesc& d = g.d;
    if (d.n_slots == 0 || d.n_slots > 8) return "n_slots must be 1..8";
    if (d.n_prof == 0 || d.n_prof > 15) return "n_prof must be 1..15";
    for (uint32_t p = 0; p < d.n_prof; ++p) {
        if (d.prof_len[p] == 0 || d.prof_nstart[p] > 8) return "bad profile";
        for (uint32_t k = 0; k < d.prof_nstart[p]; ++k) {
            if (d.prof_start[p][k] + d.prof_len[p] > d.n_slots) return "placement exceeds slots";
            g.pl.push_back({(int)p, (int)d.prof_start[p][k], (int)d.prof_len[p]});
        }
    }
    std::deque<int> todo;
    g.states.push_back({});
    g.index[{}] = 0;
    todo.push_back(0);
    while (!todo.empty()) {
        int s = todo.front();
        todo.pop_front();
        std::vector<int> out;
        for (int q = 0; q < (int)g.pl.size(); ++q) {
            if (!can_add(g, g.states[s], q)) continue;
            std::vector<int> t = with(g.states[s], q);
            auto it = g.index.find(t);
            int tid;
            if (it == g.index.end()) {
                tid = (int)g.states.size();
                g.index[t] = tid;
                g.states.push_back(t);
                todo.push_back(tid);
                if (g.states.size() > 1000000) return "state-space cap exceeded";
            } else {
                tid = it->second;
            }
            if (std::find(out.begin(), out.end(), tid) == out.end()) out.push_back(tid);
        }
        if ((int)g.succ.size() <= s) g.succ.resize(s + 1);
        g.succ[s] = out;
    }
    g.succ.resize(g.states.size());
    g.final_id.assign(g.states.size(), -1);
    for (size_t s = 0; s < g.states.size(); ++s)
        if (g.succ[s].empty()) g.final_id[s] = (int)g.n_finals++;
    // memoised reachable-final sets
    std::vector<std::vector<char>> reach(g.states.size());
    std::vector<char> done(g.states.size(), 0);
    // states only grow along alloc edges, so process in decreasing size (reverse topological order)
    std::vector<int> order(g.states.size());
    for (size_t i = 0; i < order.size(); ++i) order[i] = (int)i;
    std::sort(order.begin(), order.end(),
              [&](int a, int b) { return g.states[a].size() > g.states[b].size(); });
    for (int s : order) {
        reach[s].assign(g.n_finals, 0);
        if (g.final_id[s] >= 0) reach[s][g.final_id[s]] = 1;
        for (int t : g.succ[s]) {
            if (!done[t]) return "internal: topological order";
            for (uint32_t f = 0; f < g.n_finals; ++f) reach[s][f] |= reach[t][f];
        }
        done[s] = 1;
    }
    g.fcr.assign(g.states.size(), 0);
    for (size_t s = 0; s < g.states.size(); ++s)
        for (uint32_t f = 0; f < g.n_finals; ++f) g.fcr[s] += reach[s][f];
    // Scheme A layouts: valid states whose slices all have the level's memory
    std::vector<uint32_t> mems;
    for (uint32_t p = 0; p < d.n_prof; ++p)
        if (std::find(mems.begin(), mems.end(), g.mem(p)) == mems.end()) mems.push_back(g.mem(p));
    std::sort(mems.begin(), mems.end());
    for (size_t l = 0; l < mems.size() && l < 8; ++l) {
        std::vector<int> st;
        for (uint32_t i = 0; i < d.n_alay[l]; ++i) {
            int q = g.placement_id((int)d.alay_prof[l][i], (int)d.alay_start[l][i]);
            if (q < 0 || !can_add(g, st, q) || g.mem((int)d.alay_prof[l][i]) != mems[l]) return "scheme A layout invalid";
            st = with(st, q);
        }
    }
    // static layout must be a valid state
    std::vector<int> lay;
    for (uint32_t i = 0; i < d.n_layout; ++i) {
        int q = g.placement_id((int)d.layout_prof[i], (int)d.layout_start[i]);
        if (q < 0 || !can_add(g, lay, q)) return "static layout invalid";
        lay = with(lay, q);
    }
    return "";
}

// ---------------------------------------------------------------------------------------------------------------
// Instances (the partition manager's view) and Algorithm 2.
// ---------------------------------------------------------------------------------------------------------------
struct Instance {
    int prof, start;
    bool busy;
    int job;
    uint32_t run_start;
    // PCIe contention (flag F_PCIE, reading R39): the run in progress is re-timed whenever the number of
    // transferring runs changes. D = nominal duration (ticks), W = remaining work in 2^-16 nominal ticks since tk.
    bool started = false;
    uint32_t D = 0, end = 0, tk = 0, kind_order = 0, iters_run = 0;
    int64_t W = 0;
    uint64_t memsum = 0;  // physical MiB summed over the iterations the run executes (nominal)
};

std::vector<int> state_key(const Geometry& g, const std::vector<Instance>& inst) {
    std::vector<int> s;
    for (const Instance& i : inst) s.push_back(g.placement_id(i.prof, i.start));
    std::sort(s.begin(), s.end());
    return s;
}

uint32_t fcr_of(const Geometry& g, const std::vector<int>& key) {
    auto it = g.index.find(key);
    return it == g.index.end() ? 0u : g.fcr[it->second];
}

// allocate_partition(s, x, fcr): C <- enumerate_placements(s, x); FAIL if C = {} ; s* <- argmax_{t in C} fcr[t].
// Equal fcr: highest start slot (R5). Returns the start slot or -1 (FAIL).
int allocate_partition(const Geometry& g, const std::vector<Instance>& inst, int x) {
    std::vector<int> s = state_key(g, inst);
    int best_start = -1;
    uint32_t best_fcr = 0;
    for (int q = 0; q < (int)g.pl.size(); ++q) {
        if (g.pl[q].prof != x || !can_add(g, s, q)) continue;
        uint32_t f = fcr_of(g, with(s, q));
        if (best_start < 0 || f > best_fcr || (f == best_fcr && g.pl[q].start > best_start)) {
            best_fcr = f;
            best_start = g.pl[q].start;
        }
    }
    return best_start;
}

// ---------------------------------------------------------------------------------------------------------------
// Algorithm 3, PeakMemoryPrediction, with readings R18-R24, R37.
// ---------------------------------------------------------------------------------------------------------------
double i128_to_double(__int128 x) {  // canonical: sign-magnitude, hi*2^64 + lo
    bool neg = x < 0;
    unsigned __int128 m = neg ? (unsigned __int128)(-x) : (unsigned __int128)x;
    uint64_t hi = (uint64_t)(m >> 64), lo = (uint64_t)m;
    volatile double dh = (double)hi * 18446744073709551616.0;
    volatile double dl = (double)lo;
    double d = dh + dl;
    return neg ? -d : d;
}

struct Fit {            // result of fit_mem_model + fit_ratio + predict_peak_mem at one n
    int64_t P;          // predicted peak physical MiB incl. workspace and context (integer, R37)
    double phi, a, sigma;
};

// fit_mem_model / fit_ratio: ordinary least squares m_t = a*t + b over t = 1..n, written with the
// exact integer sums of the n samples (R18); sigma = sqrt(SSR/(n-2)) (R19).
// predict_peak_mem: mem_pred = a*T + b + z*sigma at the final iteration T = max_iter (R23),
// physical = requested / inverse-reuse forecast (R21, R22), + workspace + context
// (PAPER.md:341, :359-362).
Fit fit_and_predict(const std::vector<uint32_t>& req_mem_list, const std::vector<uint32_t>& reuse_list, uint32_t T,
                    const OrPolicy& pol, uint32_t ws) {
    const int64_t n = (int64_t)req_mem_list.size();
    int64_t Sy = 0, Sty = 0, Syy = 0, Sq = 0, Stq = 0;
    for (int64_t i = 1; i <= n; ++i) {  // sums recomputed from the lists every iteration (plain)
        int64_t y = req_mem_list[i - 1], q = reuse_list[i - 1];
        Sy += y;
        Sty += i * y;
        Syy += y * y;
        Sq += q;
        Stq += i * q;
    }
    // Closed-form OLS with x = 1..n:  a = 6K / (n(n^2-1)),  K = 2*Sum(t*y) - (n+1)*Sum(y);
    // a*T + b = [Sy(n^2-1) + 3K(2T-n-1)] / [n(n^2-1)];  SSR * n(n^2-1) = (n^2-1)(n*Syy - Sy^2) - 3K^2.
    const int64_t D = n * (n * n - 1);
    const int64_t Ky = 2 * Sty - (n + 1) * Sy;
    const int64_t Kq = 2 * Stq - (n + 1) * Sq;
    const int64_t h = 2 * (int64_t)T - n - 1;
    __int128 numY = (__int128)Sy * (n * n - 1) + (__int128)3 * Ky * h;
    __int128 ssrN = (__int128)(n * n - 1) * ((__int128)n * Syy - (__int128)Sy * Sy) - (__int128)3 * Ky * Ky;
    __int128 numQ = (__int128)Sq * (n * n - 1) + (__int128)3 * Kq * h;
    Fit f;
    double den = (double)D;
    double yT = i128_to_double(numY) / den;                                // a*T + b
    double var = i128_to_double(ssrN) / (double)(D * (n - 2));            // sigma^2
    f.sigma = std::sqrt(var);
    volatile double zs = pol.z * f.sigma;                                 // no FMA contraction
    double u = yT + zs;                                                   // mem_pred = a*T + b + z*sigma
    if (u < 0.0) u = 0.0;
    double V;
    if (pol.flags & F_EWMA) {  // R36 (north_star only; not in the paper): EWMA of the inverse reuse ratio
        int64_t L = reuse_list[0];
        for (int64_t i = 2; i <= n; ++i) L = L + (((int64_t)reuse_list[i - 1] - L) >> 3);
        V = (double)L / 65536.0;
    } else {
        V = (i128_to_double(numQ) / den) / 65536.0;                       // inverse reuse at T (Q16 -> real)
    }
    if (V < 1.0) V = 1.0;
    f.phi = u / V;
    f.a = (double)(6 * Ky) / den;
    f.P = (int64_t)std::ceil(f.phi) + (int64_t)ws + (int64_t)pol.ctx_mib;
    return f;
}

// converge(mem_pred): the last conv_k successive predictions each changed by less than
// eps_num/eps_den relative to their predecessor (R24).
bool converge(const std::vector<int64_t>& history, const OrPolicy& pol) {
    if (history.size() < (size_t)pol.conv_k + 1) return false;
    for (size_t m = history.size() - pol.conv_k; m < history.size(); ++m) {
        int64_t prev = history[m - 1], cur = history[m];
        int64_t diff = cur > prev ? cur - prev : prev - cur;
        if (!((int64_t)pol.eps_den * diff < (int64_t)pol.eps_num * prev)) return false;
    }
    return true;
}

// PeakMemoryPrediction(): for each iteration append req_mem and reuse, refit, predict at
// max_iter, return on convergence. Predictions start at n = min_n (sigma needs n >= 3, R24).
void peak_memory_prediction(const std::vector<uint32_t>& y, const std::vector<uint32_t>& q, uint32_t T,
                            const OrPolicy& pol, uint32_t ws, OrEstimate* e) {
    std::vector<uint32_t> req_mem_list, reuse_ratio_list;
    std::vector<int64_t> history;
    e->conv_iter = 0;
    e->pred_mib = 0;
    e->phi = e->a = e->sigma = 0.0;
    for (uint32_t n = 1; n <= T; ++n) {
        req_mem_list.push_back(y[n - 1]);
        reuse_ratio_list.push_back(q[n - 1]);
        if (n < pol.min_n) continue;
        Fit f = fit_and_predict(req_mem_list, reuse_ratio_list, T, pol, ws);
        history.push_back(f.P);
        e->phi = f.phi;
        e->a = f.a;
        e->sigma = f.sigma;
        if (converge(history, pol)) {
            e->conv_iter = (uint16_t)n;
            e->pred_mib = (uint32_t)f.P;
            return;
        }
    }
}

// ---------------------------------------------------------------------------------------------------------------
// Jobs: memory estimation and the workload truth the simulator checks against.
// ---------------------------------------------------------------------------------------------------------------
struct Job {
    uint32_t cls, iters, ticks, est, tru, ws, warps;
    uint32_t xfer;               // PCIe transfer fraction of an iteration, in 1/256 (record bits 24-31, R39)
    uint32_t arrival = 0;        // arrival tick (R40; 0 = batch)
    uint32_t b, q0, slope_q8, sigma, qslope;
    std::vector<uint32_t> y, q;  // DYNAMIC samples i = 1..T
    OrEstimate e;
    uint32_t req;                // current memory requirement (MiB)
};

std::vector<uint32_t> levels(const Geometry& g) {
    std::vector<uint32_t> L;
    for (uint32_t p = 0; p < g.d.n_prof; ++p)
        if (std::find(L.begin(), L.end(), g.mem(p)) == L.end()) L.push_back(g.mem(p));
    std::sort(L.begin(), L.end());
    return L;
}

// Physical memory of a job at iteration i (allocated + CUDA context decides OOM).
uint64_t physical(const Job& j, uint32_t i, const OrPolicy& pol) {
    if (j.cls == TG_CLASS_DYNAMIC)
        return (uint64_t)j.y[i - 1] * 65536u / j.q[i - 1] + j.ws + pol.ctx_mib;  // physical = req / inv_reuse (R22)
    return (uint64_t)j.tru + j.ws + pol.ctx_mib;
}

// Sum of the physical memory over iterations 1..k.
uint64_t memory_sum(const Job& j, uint32_t k, const OrPolicy& pol) {
    uint64_t s = 0;
    for (uint32_t i = 1; i <= k; ++i) s += physical(j, i, pol);
    return s;
}

// First iteration (1..T) whose physical memory exceeds cap (R12); NEVER if none.
uint16_t first_exceed(const Job& j, uint64_t cap, const OrPolicy& pol) {
    for (uint32_t i = 1; i <= j.iters; ++i)
        if (physical(j, i, pol) > cap) return (uint16_t)i;
    return NEVER;
}

struct Recorded {  // recorded per-iteration samples of one job, or none
    const uint32_t* pairs = nullptr;  // (req_mib, inv_reuse_q16) per iteration
    uint64_t count = 0;
};

Job load_job(const Geometry& g, const uint32_t* rec, const uint32_t* ext, uint64_t seed, uint64_t trace,
             uint32_t jidx, const OrPolicy& pol, Recorded rs = Recorded()) {
    Job j;
    j.cls = (rec[2] >> 16) & 0xFF;
    j.iters = rec[2] & 0xFFFF;
    j.xfer = rec[2] >> 24;
    j.ticks = rec[3];
    j.ws = ext ? ext[0] : 0;
    j.warps = ext ? ext[1] : 0;
    memset(&j.e, 0, sizeof(j.e));
    std::vector<uint32_t> L = levels(g);
    j.e.n_levels = (uint16_t)L.size();
    for (int l = 0; l < 6; ++l) j.e.fe[l] = NEVER;
    if (j.cls == TG_CLASS_DYNAMIC) {
        j.b = rec[0];
        j.q0 = rec[1];
        j.slope_q8 = ext ? ext[2] : 0;
        j.sigma = ext ? (ext[3] & 0xFFFF) : 0;
        j.qslope = ext ? (ext[3] >> 16) : 0;
        uint64_t key = tg_key(seed, trace, jidx);
        j.y.resize(j.iters);
        j.q.resize(j.iters);
        for (uint32_t i = 1; i <= j.iters; ++i) {
            if (rs.pairs && rs.count > 0) {  // recorded series (a short one repeats its last sample; flagged on GPU)
                uint64_t k = (i <= rs.count ? i : rs.count) - 1;
                j.y[i - 1] = rs.pairs[2 * k];
                j.q[i - 1] = rs.pairs[2 * k + 1];
            } else {
                tg_dyn_sample(key, i, j.b, j.slope_q8, j.sigma, j.q0, j.qslope, &j.y[i - 1], &j.q[i - 1]);
            }
        }
        // Grow-on-demand: start in the smallest partition (R16).
        j.e.req0_mib = g.mem(0);
        peak_memory_prediction(j.y, j.q, j.iters, pol, j.ws, &j.e);
    } else {
        j.est = rec[0];
        j.tru = rec[1];
        // Compile-time / model-size estimate + workspace + context.
        j.e.req0_mib = j.est + j.ws + pol.ctx_mib;
    }
    for (size_t l = 0; l < L.size() && l < 6; ++l) j.e.fe[l] = first_exceed(j, L[l], pol);
    // memory integrals over the first k iterations (PAPER.md:675 memory utilisation)
    for (size_t l = 0; l < L.size() && l < 5; ++l)
        if (j.e.fe[l] != NEVER) j.e.mem_fe[l] = (uint32_t)memory_sum(j, j.e.fe[l], pol);
    j.e.mem_conv = (uint32_t)memory_sum(j, j.e.conv_iter, pol);
    j.e.mem_T = (uint32_t)memory_sum(j, j.iters, pol);
    j.req = j.e.req0_mib;
    return j;
}

// Tight fit: smallest-memory profile holding the requirement; with warp folding, one
// whose wave count equals the full GPU's (R30); ties -> fewer compute slices (profiles are listed in that order).
int tight_fit(const Geometry& g, uint32_t req, uint32_t warps, const OrPolicy& pol) {
    int full = (int)g.d.n_prof - 1;
    for (uint32_t p = 0; p < g.d.n_prof; ++p) {
        if (g.mem(p) < req) continue;
        if ((pol.flags & F_WARP_FOLD) && warps > 0) {
            uint64_t cap_p = (uint64_t)g.d.sms_per_slice * g.d.prof_compute[p] * g.d.warps_per_sm;
            uint64_t cap_f = (uint64_t)g.d.sms_per_slice * g.d.prof_compute[full] * g.d.warps_per_sm;
            if ((warps + cap_p - 1) / cap_p != (warps + cap_f - 1) / cap_f) continue;
        }
        return (int)p;
    }
    return -1;
}

// ---------------------------------------------------------------------------------------------------------------
// The scheduler + partition manager event loop (Alg. 4).
// ---------------------------------------------------------------------------------------------------------------
struct Event {
    uint32_t tick, kind_order, job;  // kind order: COMPLETE 0 < OOM 1 < PREEMPT 2 (R28)
    bool operator>(const Event& o) const {
        if (tick != o.tick) return tick > o.tick;
        if (kind_order != o.kind_order) return kind_order > o.kind_order;
        return job > o.job;
    }
};

struct Sim {
    const Geometry& g;
    const OrPolicy& pol;
    std::vector<Job>& jobs;
    std::vector<Instance> inst;
    std::deque<int> queue;
    std::priority_queue<Event, std::vector<Event>, std::greater<Event>> events;
    OrResult r;
    uint32_t t = 0;
    size_t next_arrival = 0;  // R40: jobs [0, next_arrival) have arrived (arrival ticks are non-decreasing)
    std::vector<uint64_t>* rec_out;
    std::string err;

    Sim(const Geometry& g_, const OrPolicy& p_, std::vector<Job>& j_, std::vector<uint64_t>* ro)
        : g(g_), pol(p_), jobs(j_), rec_out(ro) {
        memset(&r, 0, sizeof(r));
        r.decision_hash = 0xcbf29ce484222325ull;
    }

    // Decision record and FNV-1a-64 hash (SURVEY.md §8(c) "Decision record and hash").
    void record(uint32_t tick, uint32_t job, uint32_t kind, uint32_t start, uint32_t prof, uint32_t nd) {
        uint64_t rec = ((uint64_t)tick << 32) | ((uint64_t)(job & 0xFFFF) << 16) | ((kind & 0xF) << 12) |
                       ((start & 0xF) << 8) | ((prof & 0xF) << 4) | (nd & 0xF);
        r.decision_hash = (r.decision_hash ^ rec) * 0x100000001b3ull;
        if (rec_out) rec_out->push_back(rec);
    }

    int find_instance(int start) {
        for (size_t i = 0; i < inst.size(); ++i)
            if (inst[i].start == start) return (int)i;
        return -1;
    }

    bool any_busy() const {
        for (const Instance& i : inst)
            if (i.busy) return true;
        return false;
    }

    // Invariants: no two instances overlap; sum of memory <= capacity; sum of compute <= GPU.
    void check_invariants() {
        uint32_t mem = 0, comp = 0;
        for (size_t a = 0; a < inst.size(); ++a) {
            mem += g.mem(inst[a].prof);
            comp += g.d.prof_compute[inst[a].prof];
            for (size_t b = a + 1; b < inst.size(); ++b) {
                Placement pa{inst[a].prof, inst[a].start, (int)g.d.prof_len[inst[a].prof]};
                Placement pb{inst[b].prof, inst[b].start, (int)g.d.prof_len[inst[b].prof]};
                if (overlaps(pa, pb)) err = "invariant: overlapping instances";
            }
        }
        if (mem > g.full_mem()) err = "invariant: memory over capacity";
        if (comp > g.d.n_compute) err = "invariant: compute over capacity";
    }

    // Start a run of job j on instance k. Created instances start after reconfig_ticks (R27).
    void start_run(int jid, int k, bool created) {
        Instance& in = inst[k];
        Job& j = jobs[jid];
        in.busy = true;
        in.job = jid;
        uint32_t s = t + (created ? pol.reconfig_ticks : 0);
        in.run_start = s;
        uint32_t cap = pol.kind == BASELINE ? g.full_mem() : g.mem(in.prof);
        uint32_t T = j.iters;
        // Iteration time on the slice (R31 variant, flag WAVE_TIME): iter_ticks are full-GPU times; a job of W warps
        // needs waves(W, p) = ceil(W / (sms_per_slice * compute(p) * warps_per_sm)) waves, so an
        // iteration takes ceil(ticks * waves(W, p) / waves(W, full)) ticks on profile p.
        uint32_t ticks = j.ticks;
        if ((pol.flags & F_WAVE_TIME) && j.warps > 0) {
            uint64_t cp = (uint64_t)g.d.sms_per_slice * g.d.prof_compute[in.prof] * g.d.warps_per_sm;
            uint64_t cf = (uint64_t)g.d.sms_per_slice * g.d.prof_compute[g.d.n_prof - 1] * g.d.warps_per_sm;
            uint64_t wp = (j.warps + cp - 1) / cp, wf = (j.warps + cf - 1) / cf;
            ticks = (uint32_t)(((uint64_t)j.ticks * wp + wf - 1) / wf);
        }
        // OOM at the end of the first iteration whose physical memory exceeds the slice (R12).
        uint32_t i_oom = first_exceed(j, cap, pol);
        // Early restart (R25): converged forecast above the slice, and a larger slice exists.
        uint32_t i_pre = 0xFFFFFFFFu;
        if ((pol.flags & F_EARLY_RESTART) && pol.kind != BASELINE && j.cls == TG_CLASS_DYNAMIC &&
            j.e.conv_iter > 0 && j.e.pred_mib > cap && cap < g.full_mem())
            i_pre = j.e.conv_iter;
        Event ev;
        ev.job = (uint32_t)jid;
        uint32_t end;
        // Same-iteration precedence OOM > COMPLETE > PREEMPT (R29).
        if (i_oom != NEVER && i_oom <= std::min(T, i_pre)) {
            ev.kind_order = 1;
            end = s + i_oom * ticks;
        } else if (i_pre < T) {
            ev.kind_order = 2;
            end = s + i_pre * ticks;
        } else {
            ev.kind_order = 0;
            end = s + T * ticks;
        }
        ev.tick = end;
        uint32_t comp = pol.kind == BASELINE ? g.d.n_compute : g.d.prof_compute[in.prof];
        // memory held while running: iterations 1..k at `ticks` each (k = OOM / preempt / last iteration)
        uint32_t iters_run = ev.kind_order == 1 ? i_oom : ev.kind_order == 2 ? i_pre : T;
        if (pol.flags & F_PCIE) {  // R39: the end is known only as the run progresses (retime, run_pcie)
            in.started = false;
            in.D = end - s;
            in.kind_order = ev.kind_order;
            in.iters_run = iters_run;
            in.memsum = memory_sum(j, iters_run, pol);
            return;
        }
        r.busy_slice_ticks += (uint64_t)comp * (end - s);
        r.mem_mib_ticks += memory_sum(j, iters_run, pol) * ticks;
        if (ev.kind_order != 0) r.wasted_ticks += end - s;
        events.push(ev);
    }

    // ---- PCIe contention ("PCIe bandwidth remains a shared resource, being equally divided among
    // multiple MIG instances"; reading R39) ----
    // A run of a job with transfer fraction F/256 > 0 shares PCIe with the other transferring runs in progress
    // (c of them): its transfer time is multiplied by c, its kernel time is not, so it advances at
    // 2^24 / (256 - F + F c) units of 2^-16 nominal ticks per tick (floor). Runs with F = 0 are unaffected.
    uint32_t c_eff = 0;  // transferring runs in progress since the last retime

    static int64_t rate(uint32_t F, uint32_t c) {
        return F == 0 ? 65536 : (int64_t)((1u << 24) / (256u - F + F * c));
    }

    // Every run in progress advances from its last retime tick to t at the concurrency in effect (c_eff).
    void advance(uint32_t tt) {
        for (Instance& in : inst)
            if (in.busy && in.started) {
                in.W -= (int64_t)(tt - in.tk) * rate(jobs[in.job].xfer, c_eff);
                in.tk = tt;
            }
    }

    // At tick t, after the events and the scheduler pass: runs due to start now begin (full nominal work), the
    // concurrency is recounted and every run in progress gets its end for the new rate.
    void retime() {
        uint32_t c = 0;
        for (Instance& in : inst) {
            if (!in.busy) continue;
            if (!in.started && in.run_start == t) {
                in.started = true;
                in.tk = t;
                in.W = (int64_t)in.D << 16;
            }
            if (in.started && jobs[in.job].xfer > 0) ++c;
        }
        for (Instance& in : inst)
            if (in.busy && in.started) {
                const int64_t rho = rate(jobs[in.job].xfer, c);
                in.end = t + (uint32_t)((in.W + rho - 1) / rho);
            }
        c_eff = c;
    }

    // A run ends at t: its actual duration counts for power, memory and waste (R26, R39).
    void end_run(int k) {
        Instance& in = inst[k];
        const Job& j = jobs[in.job];
        const uint32_t actual = t - in.run_start;
        const uint32_t comp = pol.kind == BASELINE ? g.d.n_compute : g.d.prof_compute[in.prof];
        r.busy_slice_ticks += (uint64_t)comp * actual;
        // memory: a constant footprint for the whole run; a DYNAMIC job's iterations stretched uniformly
        r.mem_mib_ticks += j.cls == TG_CLASS_DYNAMIC ? (in.iters_run ? in.memsum * actual / in.iters_run : 0)
                                                     : physical(j, 1, pol) * actual;
        if (in.kind_order != 0) r.wasted_ticks += actual;
        Event ev;
        ev.tick = t;
        ev.kind_order = in.kind_order;
        ev.job = (uint32_t)in.job;
        apply(ev);
    }

    // The event loop with re-timing: the next tick is the earliest end or pending start; ends are applied in R28
    // order and followed by one scheduler pass; a tick with only starts has no pass (nothing finished).
    void run_pcie(bool scheme_a) {
        retime();
        for (;;) {
            uint32_t tn = next_arrival_tick();
            for (const Instance& in : inst)
                if (in.busy) tn = std::min(tn, in.started ? in.end : in.run_start);
            if (tn == 0xFFFFFFFFu) break;
            advance(tn);
            t = tn;
            std::vector<std::pair<uint64_t, int>> ends;  // (kind order, job) -> instance
            for (size_t k = 0; k < inst.size(); ++k)
                if (inst[k].busy && inst[k].started && inst[k].end == t)
                    ends.push_back({((uint64_t)inst[k].kind_order << 32) | (uint32_t)inst[k].job, inst[k].start});
            std::sort(ends.begin(), ends.end());
            for (auto& e : ends) end_run(find_instance(e.second));
            const bool arrived = !scheme_a && admit_arrivals();
            if (!ends.empty() || arrived) r.makespan = t;
            if (!ends.empty() || arrived) {
                if (scheme_a) a_step();
                else scheduler_pass();
            }
            retime();
            check_invariants();
            if (!err.empty()) return;
        }
    }

    // One scheduler pass at tick t (Alg. 4; wake on every event, R9).
    void scheduler_pass() {
        while (!queue.empty()) {
            int jid = queue.front();
            Job& j = jobs[jid];
            int need = tight_fit(g, j.req, j.warps, pol);
            if (need < 0) {  // no profile can ever hold the job
                record(t, jid, K_REJECT, 0xF, 0xF, 0);
                r.rejected++;
                queue.pop_front();
                continue;
            }
            uint32_t need_mem = g.mem(need), need_comp = g.d.prof_compute[need];
            if (pol.kind == BASELINE) {  // one job at a time on the non-partitioned GPU
                if (any_busy()) {
                    record(t, jid, K_WAIT, 0xF, need, 0);
                    r.waits++;
                    return;
                }
                int k = find_instance(0);
                record(t, jid, K_PLACE_BASELINE, 0, inst[k].prof, 0);
                r.placements++;
                queue.pop_front();
                start_run(jid, k, false);
                continue;
            }
            if (pol.kind == STATIC) {  // fixed slices (R11)
                int best = -1;
                bool could = false;
                for (size_t k = 0; k < inst.size(); ++k) {
                    if (g.mem(inst[k].prof) < need_mem || g.d.prof_compute[inst[k].prof] < need_comp) continue;
                    could = true;
                    if (inst[k].busy) continue;
                    if (best < 0 || g.mem(inst[k].prof) < g.mem(inst[best].prof) ||
                        (g.mem(inst[k].prof) == g.mem(inst[best].prof) && inst[k].start > inst[best].start))
                        best = (int)k;
                }
                if (best >= 0) {
                    record(t, jid, K_PLACE_STATIC, inst[best].start, inst[best].prof, 0);
                    r.placements++;
                    queue.pop_front();
                    start_run(jid, best, false);
                    continue;
                }
                if (could) {
                    record(t, jid, K_WAIT, 0xF, need, 0);
                    r.waits++;
                    return;
                }
                record(t, jid, K_REJECT, 0xF, need, 0);
                r.rejected++;
                queue.pop_front();
                continue;
            }
            if (pol.kind == FUSION_FISSION) {
                // try_schedule(j): an idle partition that tightly fits (R7).
                int best = -1;
                for (size_t k = 0; k < inst.size(); ++k) {
                    if (inst[k].busy || g.mem(inst[k].prof) != need_mem ||
                        g.d.prof_compute[inst[k].prof] < need_comp)
                        continue;
                    if (best < 0 || inst[k].start > inst[best].start) best = (int)k;
                }
                if (best >= 0) {
                    record(t, jid, K_REUSE, inst[best].start, inst[best].prof, 0);
                    r.placements++;
                    queue.pop_front();
                    start_run(jid, best, false);
                    continue;
                }
            }
            // try_new_mig_slice(j.memfp) -> allocate_partition (Alg. 2).
            int st = allocate_partition(g, inst, need);
            if (st >= 0) {
                inst.push_back({need, st, false, -1, 0});
                r.creates++;
                check_invariants();
                record(t, jid, K_ALLOC, st, need, 0);
                r.placements++;
                queue.pop_front();
                start_run(jid, (int)inst.size() - 1, true);
                continue;
            }
            if (pol.kind == FUSION_FISSION) {
                // Fusion / fission (R8): for each placement q of the profile whose overlapping
                // instances are all idle (at least one), destroy them and create q. Best (fcr, -#destroyed, start).
                int best_q = -1, best_nd = 0;
                uint32_t best_f = 0;
                for (int q = 0; q < (int)g.pl.size(); ++q) {
                    if (g.pl[q].prof != need) continue;
                    bool ok = true;
                    int nd = 0;
                    std::vector<Instance> keep;
                    for (const Instance& in : inst) {
                        Placement p{in.prof, in.start, (int)g.d.prof_len[in.prof]};
                        if (overlaps(p, g.pl[q])) {
                            if (in.busy) ok = false;
                            nd++;
                        } else {
                            keep.push_back(in);
                        }
                    }
                    if (!ok || nd == 0) continue;
                    std::vector<int> key = state_key(g, keep);
                    if (!can_add(g, key, q)) continue;
                    uint32_t f = fcr_of(g, with(key, q));
                    bool better = best_q < 0 || f > best_f || (f == best_f && nd < best_nd) ||
                                  (f == best_f && nd == best_nd && g.pl[q].start > g.pl[best_q].start);
                    if (better) {
                        best_q = q;
                        best_f = f;
                        best_nd = nd;
                    }
                }
                if (best_q >= 0) {
                    std::vector<Instance> keep;
                    for (const Instance& in : inst) {
                        Placement p{in.prof, in.start, (int)g.d.prof_len[in.prof]};
                        if (!overlaps(p, g.pl[best_q])) keep.push_back(in);
                    }
                    inst = keep;
                    r.destroys += best_nd;
                    inst.push_back({need, g.pl[best_q].start, false, -1, 0});
                    r.creates++;
                    check_invariants();
                    record(t, jid, K_RECONF, g.pl[best_q].start, need, best_nd);
                    r.placements++;
                    queue.pop_front();
                    start_run(jid, (int)inst.size() - 1, true);
                    continue;
                }
            }
            // sleep() until a running job finishes; head-of-line.
            record(t, jid, K_WAIT, 0xF, need, 0);
            r.waits++;
            return;
        }
    }

    // Arrival streams (reading R40): every job whose arrival tick is <= t joins the queue tail, in queue order,
    // after the requeues of the events at t. Returns whether any arrived.
    bool admit_arrivals() {
        bool any = false;
        while (next_arrival < jobs.size() && jobs[next_arrival].arrival <= t) {
            queue.push_back((int)next_arrival++);
            any = true;
        }
        return any;
    }
    uint32_t next_arrival_tick() const {
        return next_arrival < jobs.size() ? jobs[next_arrival].arrival : 0xFFFFFFFFu;
    }

    // Next-larger slice after an OOM (R14): smallest profile memory strictly above cap.
    bool next_larger(uint32_t cap, uint32_t* out) {
        for (uint32_t p = 0; p < g.d.n_prof; ++p)
            if (g.mem(p) > cap) {
                *out = g.mem(p);
                return true;
            }
        return false;
    }

    void requeue(int jid) {
        if (pol.kind == SCHEME_A)
            a_enqueue(jid);  // the tail of its new (larger) group
        else
            queue.push_back(jid);
    }

    void apply(const Event& ev) {
        int k = -1;
        for (size_t i = 0; i < inst.size(); ++i)
            if (inst[i].busy && inst[i].job == (int)ev.job) k = (int)i;
        if (k < 0) {
            err = "internal: event without instance";
            return;
        }
        Instance& in = inst[k];
        Job& j = jobs[ev.job];
        uint32_t cap = pol.kind == BASELINE ? g.full_mem() : g.mem(in.prof);
        if (ev.kind_order == 0) {
            record(t, ev.job, K_COMPLETE, in.start, in.prof, 0);
            r.completed++;
            r.turnaround_sum += t - j.arrival;  // completion - arrival (R34: batch, all 0; R40: streams)
        } else if (ev.kind_order == 1) {
            record(t, ev.job, K_OOM, in.start, in.prof, 0);
            r.ooms++;
            uint32_t nl;
            if (next_larger(cap, &nl)) {
                j.req = nl;
                r.restarts++;
                requeue((int)ev.job);  // return to the scheduling queue, at the tail (R13)
            } else {
                record(t, ev.job, K_FAILED, in.start, in.prof, 0);
                r.failed++;
            }
        } else {
            record(t, ev.job, K_PREEMPT, in.start, in.prof, 0);
            r.preempts++;
            r.restarts++;
            j.req = std::min(j.e.pred_mib, g.full_mem());  // restart on the slice meeting the forecast (R25)
            requeue((int)ev.job);
        }
        in.busy = false;
        in.job = -1;
        if (pol.kind == DYNAMIC) {  // create on demand, free on completion (R10)
            inst.erase(inst.begin() + k);
            r.destroys++;
        }
    }

    // ---- Scheme A, schedule_by_group (Alg. PAPER.md:583-595; reading R38) ----
    // Jobs are grouped by the memory of their tight-fit profile; groups run in ascending memory order on that
    // group's homogeneous layout; job k of a group goes to slice (k mod #slices) (static round robin over slices
    // in ascending start) and each slice runs its jobs in order. The GPU is reconfigured only when a
    // group has drained. OOM'd / preempted jobs join the tail of their new (larger) group.
    struct GroupState {
        std::vector<std::vector<int>> lists;  // per level: job ids in group order
        int cur = -1;
        std::vector<size_t> next_idx;         // per slice of the current layout
        std::vector<uint32_t> ready;          // per slice: earliest start (after creation)
    };
    GroupState gs;

    int level_of_prof(int p) const {
        std::vector<uint32_t> L = levels(g);
        return (int)(std::find(L.begin(), L.end(), g.mem(p)) - L.begin());
    }

    void a_enqueue(int jid) {
        Job& j = jobs[jid];
        int need = tight_fit(g, j.req, j.warps, pol);
        if (need < 0) {  // cannot happen after an OOM/preempt (the new requirement always fits the GPU)
            record(t, jid, K_REJECT, 0xF, 0xF, 0);
            r.rejected++;
            return;
        }
        gs.lists[level_of_prof(need)].push_back(jid);
    }

    bool a_group_done() const {
        for (const Instance& in : inst)
            if (in.busy) return false;
        for (size_t k = 0; k < gs.next_idx.size(); ++k)
            if (gs.next_idx[k] < gs.lists[gs.cur].size()) return false;
        return true;
    }

    void a_dispatch() {
        for (size_t k = 0; k < inst.size(); ++k) {  // instances are kept in ascending start order
            if (inst[k].busy || gs.next_idx[k] >= gs.lists[gs.cur].size()) continue;
            int jid = gs.lists[gs.cur][gs.next_idx[k]];
            gs.next_idx[k] += inst.size();
            record(t, jid, K_PLACE_GROUP, inst[k].start, inst[k].prof, 0);
            r.placements++;
            uint32_t save = t;
            bool created = t < gs.ready[k];  // first run on a freshly created slice waits for it
            start_run(jid, (int)k, created);
            t = save;
        }
    }

    bool a_next_group() {
        int nl = -1;
        for (int l = gs.cur + 1; l < (int)gs.lists.size(); ++l)
            if (!gs.lists[l].empty()) {
                nl = l;
                break;
            }
        if (nl < 0) return false;
        uint32_t nd = (uint32_t)inst.size();
        r.destroys += nd;
        inst.clear();
        gs.cur = nl;
        std::vector<std::pair<int, int>> sl;
        for (uint32_t i = 0; i < g.d.n_alay[nl]; ++i) sl.push_back({(int)g.d.alay_start[nl][i], (int)g.d.alay_prof[nl][i]});
        std::sort(sl.begin(), sl.end());
        for (auto& e : sl) inst.push_back({e.second, e.first, false, -1, 0});
        r.creates += (uint32_t)inst.size();
        check_invariants();
        gs.next_idx.assign(inst.size(), 0);
        for (size_t k = 0; k < inst.size(); ++k) gs.next_idx[k] = k;
        gs.ready.assign(inst.size(), t + pol.reconfig_ticks);
        record(t, 0xFFFF, K_LAYOUT, 0, (uint32_t)nl, nd);
        return true;
    }

    void a_step() {  // after the events of tick t
        if (gs.cur >= 0) a_dispatch();
        while (gs.cur < 0 || a_group_done()) {
            if (!a_next_group()) return;
            a_dispatch();
        }
    }

    void run_scheme_a() {
        gs.lists.assign(levels(g).size(), {});
        t = 0;
        for (size_t i = 0; i < jobs.size(); ++i) a_enqueue((int)i);  // REJECTs at t = 0, in queue order
        next_arrival = jobs.size();                                   // the whole queue is grouped at t = 0
        a_step();
        if (pol.flags & F_PCIE) run_pcie(true);
        while (!events.empty()) {
            t = events.top().tick;
            while (!events.empty() && events.top().tick == t) {
                Event ev = events.top();
                events.pop();
                apply(ev);
            }
            r.makespan = t;
            a_step();
            check_invariants();
            if (!err.empty()) return;
        }
        r.energy_wticks = (uint64_t)pol.idle_w * r.makespan + (uint64_t)pol.w_per_slice * r.busy_slice_ticks;
    }

    void run() {
        r.n_jobs = (uint32_t)jobs.size();
        if (pol.kind == SCHEME_A) {
            run_scheme_a();
            return;
        }
        if (pol.kind == BASELINE) {
            inst.push_back({(int)g.d.n_prof - 1, 0, false, -1, 0});
        } else if (pol.kind == STATIC) {
            for (uint32_t i = 0; i < g.d.n_layout; ++i)
                inst.push_back({(int)g.d.layout_prof[i], (int)g.d.layout_start[i], false, -1, 0});
        }
        t = 0;
        admit_arrivals();
        scheduler_pass();
        if (pol.flags & F_PCIE) run_pcie(false);
        // the next tick: the earliest run end or job arrival (R9, R40)
        while (!events.empty() || next_arrival < jobs.size()) {
            t = std::min(events.empty() ? 0xFFFFFFFFu : events.top().tick, next_arrival_tick());
            while (!events.empty() && events.top().tick == t) {
                Event ev = events.top();
                events.pop();
                apply(ev);
            }
            r.makespan = t;  // the last tick with an end or an arrival (R40: a late arrival may only be rejected)
            admit_arrivals();
            scheduler_pass();
            check_invariants();
            if (!err.empty()) return;
        }
        if (!queue.empty()) err = "stall: queue non-empty with nothing running";
        r.energy_wticks = (uint64_t)pol.idle_w * r.makespan + (uint64_t)pol.w_per_slice * r.busy_slice_ticks;
    }
};

thread_local std::string g_err;

}  // namespace

extern "C" {

const char* or_last_error() { return g_err.c_str(); }

void* or_geometry_new(const OrGeomDesc* d) {
    Geometry* g = new Geometry();
    g->d = *d;
    g_err = build_geometry(*g);
    if (!g_err.empty()) {
        delete g;
        return nullptr;
    }
    return g;
}

void or_geometry_free(void* g) { delete (Geometry*)g; }

// Alg. 1 for an arbitrary slot geometry given as placement masks (bit i = memory slot i), by its
// literal definition: the valid partition states are the sets of pairwise disjoint placements (enumerated
// exhaustively), the final states those to which no placement can be added (R2), and fcr(s) = the number of final
// states that contain s (every superset of s that is a state is reached by adding its missing placements). The
// per-occupancy table fcr_out[m] (2^n_slots entries, 0 where no state has occupancy m) asserts R3: every state with
// occupancy m has the same fcr. Returns 0, -1 (more than 2 000 000 states), -2 (R3 violated), -3 (bad input).
int or_reach(uint32_t n_slots, const uint32_t* masks, uint32_t n_pl, uint32_t* fcr_out, uint64_t* n_states,
             uint64_t* n_finals) {
    if (n_slots < 1 || n_slots > 20 || n_pl < 1) return -3;
    std::vector<std::vector<int>> states;
    std::vector<uint32_t> occ;
    std::vector<int> cur;
    // every set of pairwise disjoint placements, each once (placements added in increasing index order)
    std::function<bool(int, uint32_t)> rec = [&](int from, uint32_t m) -> bool {
        states.push_back(cur);
        occ.push_back(m);
        if (states.size() > 2000000) return false;
        for (int q = from; q < (int)n_pl; ++q) {
            if (masks[q] & m) continue;
            cur.push_back(q);
            if (!rec(q + 1, m | masks[q])) return false;
            cur.pop_back();
        }
        return true;
    };
    if (!rec(0, 0u)) return -1;
    std::vector<int> finals;
    for (size_t i = 0; i < states.size(); ++i) {
        bool fits = false;
        for (uint32_t q = 0; q < n_pl && !fits; ++q) fits = (masks[q] & occ[i]) == 0;
        if (!fits) finals.push_back((int)i);
    }
    const uint32_t N = 1u << n_slots;
    std::vector<int64_t> table(N, -1);
    for (size_t i = 0; i < states.size(); ++i) {
        uint32_t c = 0;
        for (int f : finals) {  // s is a subset of F (both sorted placement lists)
            if ((occ[i] & ~occ[f]) != 0) continue;
            c += std::includes(states[f].begin(), states[f].end(), states[i].begin(), states[i].end()) ? 1u : 0u;
        }
        if (table[occ[i]] >= 0 && table[occ[i]] != (int64_t)c) return -2;
        table[occ[i]] = c;
    }
    for (uint32_t m = 0; m < N; ++m) fcr_out[m] = table[m] < 0 ? 0u : (uint32_t)table[m];
    *n_states = states.size();
    *n_finals = finals.size();
    return 0;
}

void or_geometry_counts(void* gp, uint32_t* n_states, uint32_t* n_finals, uint32_t* n_placements) {
    Geometry* g = (Geometry*)gp;
    *n_states = (uint32_t)g->states.size();
    *n_finals = g->n_finals;
    *n_placements = (uint32_t)g->pl.size();
}

// State i of S as instance lists (prof, start); returns the instance count, -1 if i out of range.
int or_geometry_state(void* gp, uint32_t i, uint32_t* prof, uint32_t* start, uint32_t* fcr, int32_t* is_final) {
    Geometry* g = (Geometry*)gp;
    if (i >= g->states.size()) return -1;
    int n = 0;
    for (int q : g->states[i]) {
        prof[n] = (uint32_t)g->pl[q].prof;
        start[n] = (uint32_t)g->pl[q].start;
        n++;
    }
    *fcr = g->fcr[i];
    *is_final = g->final_id[i] >= 0;
    return n;
}

// fcr of the state given as an instance list; 0 if not a valid state.
uint32_t or_state_fcr(void* gp, const uint32_t* prof, const uint32_t* start, uint32_t n) {
    Geometry* g = (Geometry*)gp;
    std::vector<Instance> inst;
    for (uint32_t i = 0; i < n; ++i) inst.push_back({(int)prof[i], (int)start[i], false, -1, 0});
    std::vector<int> key = state_key(*g, inst);
    for (int q : key)
        if (q < 0) return 0;
    return fcr_of(*g, key);
}

// Alg. 2 on the given state: returns the chosen start slot or -1 (FAIL).
int or_allocate(void* gp, const uint32_t* prof, const uint32_t* start, uint32_t n, uint32_t x) {
    Geometry* g = (Geometry*)gp;
    std::vector<Instance> inst;
    for (uint32_t i = 0; i < n; ++i) inst.push_back({(int)prof[i], (int)start[i], false, -1, 0});
    return allocate_partition(*g, inst, (int)x);
}

int or_tight_fit(void* gp, uint32_t req, uint32_t warps, const OrPolicy* pol) {
    return tight_fit(*(Geometry*)gp, req, warps, *pol);
}

// Alg. 3 on an explicit series y[0..T-1] (MiB), q[0..T-1] (Q16).
void or_predict_series(const uint32_t* y, const uint32_t* q, uint32_t T, const OrPolicy* pol, uint32_t ws,
                       OrEstimate* out) {
    std::vector<uint32_t> yy(y, y + T), qq(q, q + T);
    memset(out, 0, sizeof(*out));
    peak_memory_prediction(yy, qq, T, *pol, ws, out);
}

// One fit at n = len(y) (diagnostic access to fit_and_predict).
void or_fit_once(const uint32_t* y, const uint32_t* q, uint32_t n, uint32_t T, const OrPolicy* pol, uint32_t ws,
                 int64_t* P, double* phi, double* a, double* sigma) {
    std::vector<uint32_t> yy(y, y + n), qq(q, q + n);
    Fit f = fit_and_predict(yy, qq, T, *pol, ws);
    *P = f.P;
    *phi = f.phi;
    *a = f.a;
    *sigma = f.sigma;
}

// Per-job estimates for traces [0, n_traces) (trace ids trace_id0 + t).
static Recorded recorded(const uint32_t* samples, const uint64_t* sample_off, uint64_t j) {
    Recorded r;
    if (samples && sample_off) {
        r.pairs = samples + 2 * (sample_off[j] - sample_off[0]);
        r.count = sample_off[j + 1] - sample_off[j];
    }
    return r;
}

int or_estimate(void* gp, const uint32_t* jobs, const uint32_t* ext, const uint64_t* trace_off, uint64_t n_traces,
                uint64_t trace_id0, uint64_t seed, const OrPolicy* pol, OrEstimate* out, const uint32_t* samples,
                const uint64_t* sample_off) {
    Geometry* g = (Geometry*)gp;
    for (uint64_t t = 0; t < n_traces; ++t)
        for (uint64_t j = trace_off[t]; j < trace_off[t + 1]; ++j) {
            Job jb = load_job(*g, jobs + 4 * j, ext ? ext + 4 * j : nullptr, seed, trace_id0 + t,
                              (uint32_t)(j - trace_off[t]), *pol, recorded(samples, sample_off, j));
            out[j] = jb.e;
        }
    return 0;
}

// Simulate traces [t0, t1) under n_pol policies; out[(t - t0) * n_pol + p]. If rec != NULL (single trace and
// policy only), the decision records are written there (up to rec_cap) and their count to *rec_n.
int or_simulate(void* gp, const uint32_t* jobs, const uint32_t* ext, const uint64_t* trace_off, uint64_t t0,
                uint64_t t1, uint64_t trace_id0, uint64_t seed, const OrPolicy* pols, uint32_t n_pol, OrResult* out,
                uint64_t* rec, uint64_t rec_cap, uint64_t* rec_n, const uint32_t* samples,
                const uint64_t* sample_off, const uint32_t* arrival) {
    Geometry* g = (Geometry*)gp;
    g_err.clear();
    for (uint64_t t = t0; t < t1; ++t) {
        uint64_t nj = trace_off[t + 1] - trace_off[t];
        if (nj > 0xFFFF) {
            g_err = "trace has more than 65535 jobs";
            return -1;
        }
        for (uint32_t p = 0; p < n_pol; ++p) {
            std::vector<Job> js;
            for (uint64_t j = trace_off[t]; j < trace_off[t + 1]; ++j) {
                js.push_back(load_job(*g, jobs + 4 * j, ext ? ext + 4 * j : nullptr, seed, trace_id0 + t,
                                      (uint32_t)(j - trace_off[t]), pols[p], recorded(samples, sample_off, j)));
                if (arrival) {  // R40: non-decreasing within a trace
                    js.back().arrival = arrival[j];
                    if (js.size() > 1 && arrival[j] < js[js.size() - 2].arrival) {
                        g_err = "trace " + std::to_string(t) + ": arrival ticks decrease";
                        return -1;
                    }
                }
            }
            if (arrival && pols[p].kind == SCHEME_A) {
                g_err = "Scheme A groups the whole queue at t = 0: no arrival streams";
                return -1;
            }
            std::vector<uint64_t> recs;
            Sim sim(*g, pols[p], js, rec ? &recs : nullptr);
            sim.run();
            if (!sim.err.empty()) {
                g_err = "trace " + std::to_string(t) + ": " + sim.err;
                return -1;
            }
            out[(t - t0) * n_pol + p] = sim.r;
            if (rec) {
                uint64_t n = std::min<uint64_t>(recs.size(), rec_cap);
                for (uint64_t i = 0; i < n; ++i) rec[i] = recs[i];
                *rec_n = recs.size();
            }
        }
    }
    return 0;
}

}  // extern "C"
