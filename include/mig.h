/* mig.h — C ABI of libmig.so: batched simulation of the MIGM dynamic MIG partition manager + scheduler
 * (arXiv 2508.18556, "Managing Multi Instance GPUs for High Throughput and Energy Savings") over very many
 * independent synthetic job queues ("traces"), on B200 (sm_100a).
 *
 * The calls follow the paper's problem statement: jobs with a memory footprint, duration and compute need arrive at
 * a scheduler, which asks the partition manager for a slice.
 *
 *   mig_geometry_load    GPU geometry + Alg. 1 reachability table            [host]
 *   mig_estimate_memory  per-job memory estimation: compile-time / model-size estimates
 *                         and the time-series predictor Alg. 3
 *                                                                               [device, async]
 *   mig_simulate         right-sized request, Alg. 2 placement,
 *                        Scheme B + fusion/fission, OOM restart,
 *                        early restart, metrics                  [device, async]
 *   mig_simulate_host    the same from HOST buffers (H2D, estimate, simulate, D2H pipelined)       [host, sync]
 *
 * Conventions
 *   - Every entry point returns a mig_status; mig_last_error() gives a thread-local message for the last failure.
 *   - Units: time = integer ticks (1 tick = 1 ms), memory = integer MiB, power = integer W, energy = W*ticks.
 *   - Ownership: the library never frees or retains caller memory beyond a call (device calls: beyond the
 *     stream-ordered work they enqueue). A mig_geometry owns its host tables and per-device copies.
 *   - Asynchrony: device entry points are stream-ordered; outputs are valid once the stream is synchronised.
 *     Internally mig_simulate may fork work onto a library-owned side stream of the calling thread (one per thread
 *     and device, so calls from different threads never share one); it joins back into the caller's stream by
 *     events before returning, so the call stays stream-ordered and can be captured in a CUDA graph while other
 *     threads keep calling the library. Device scratch comes from a pool private to the library
 *     (mig_release_scratch).
 *   - Semantic outcomes (rejected or failed jobs) are counted in results, never reported as errors. Call errors
 *     are malformed arguments (MIG_E_INVALID_ARG), geometry problems (MIG_E_IO / PARSE / VALIDATION / CAPACITY),
 *     trace-format violations detected on the device (reported in mig_policy_totals.error_flags), and CUDA
 *     failures (MIG_E_CUDA).
 *   - No CPU fallback: without a CUDA device the device entry points fail with MIG_E_CUDA.
 *   - Determinism: results are a pure function of (geometry, traces, policies).
 */
#ifndef MIG_H
#define MIG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    MIG_OK = 0,
    MIG_E_INVALID_ARG = 1,
    MIG_E_IO = 2,
    MIG_E_PARSE = 3,
    MIG_E_VALIDATION = 4,
    MIG_E_CAPACITY = 5, /* geometry state space too large */
    MIG_E_CUDA = 6,
    MIG_E_UNSUPPORTED = 7
} mig_status;

/* Message for the last non-OK status on this thread (valid until the next call on this thread). */
const char* mig_last_error(void);

/* ------------------------------------------------------------------------------------------------------------------
 * Geometry (profiles and placement rules; Alg. 1)
 * ---------------------------------------------------------------------------------------------------------------- */
typedef struct mig_geometry mig_geometry; /* opaque; immutable after load; shareable across threads and streams */

#define MIG_MAX_SLOTS 8
#define MIG_MAX_PROFILES 15
#define MIG_MAX_LEVELS 5 /* distinct profile memory sizes */

typedef struct {
    char gpu_name[64];
    uint32_t n_slots;      /* memory slots (8 on A100/H100, 4 on A30) */
    uint32_t slot_mib;     /* MiB per memory slot */
    uint32_t n_compute;    /* compute slices of the GPU */
    uint32_t n_profiles;   /* profiles, sorted by (memory, compute) ascending */
    uint32_t n_levels;     /* distinct profile memory sizes */
    uint32_t n_placements; /* legal (profile, start) pairs */
    uint32_t n_states;     /* |S|: valid partition states (sets of placed instances) */
    uint32_t n_finals;     /* |F|: fully configured states (no legal allocation remains) */
    uint32_t fcr_s0;       /* fcr(empty GPU) */
    uint32_t full_mem_mib; /* memory of the whole GPU */
    uint32_t n_layout;     /* instances of the static layout (policy MIG_STATIC) */
    uint32_t scheme_a;     /* 1 if every memory level has a Scheme A layout (policy MIG_SCHEME_A usable) */
    uint32_t idle_w, w_per_slice; /* default power model (W idle; W per busy compute slice) */
} mig_geometry_info;

/* Load a geometry from a JSON file path, or "builtin:<name>" for the tables shipped next to libmig.so
 * (a30-24gb, a100-40gb, a100-40gb-1g10, a100-80gb, h100-80gb). Validates the placement table (every placement
 * inside the slots; profiles sorted by memory then compute; at most MIG_MAX_* of each), enumerates the valid
 * states, and builds the fcr table indexed by the occupancy bitmask (bit i = memory slot i busy).
 * Errors: MIG_E_IO (file), MIG_E_PARSE (JSON; message names the offset), MIG_E_VALIDATION (message names the
 * field), MIG_E_CAPACITY. *out is set only on MIG_OK; free with mig_geometry_free. */
mig_status mig_geometry_load(const char* json_path_or_builtin, mig_geometry** out);
void mig_geometry_free(mig_geometry* g);
mig_status mig_geometry_query(const mig_geometry* g, mig_geometry_info* out);

/* Profile p (0 <= p < n_profiles): memory MiB, compute slices, memory slots, name (<= 31 chars + NUL). */
mig_status mig_geometry_profile(const mig_geometry* g, uint32_t p, uint32_t* mem_mib, uint32_t* compute,
                                uint32_t* slots, char name[32]);

/* fcr of an occupancy mask: number of fully configured states reachable from it. 0 for masks that
 * are not the occupancy of any valid state. Host-only test hook. */
mig_status mig_geometry_fcr(const mig_geometry* g, uint32_t occ_mask, uint32_t* fcr);

/* Alg. 2 allocate_partition on an occupancy mask: the start slot of the legal placement of
 * `profile` maximising fcr (equal fcr: highest start), or -1 = FAIL. Host-only test hook. */
mig_status mig_geometry_place(const mig_geometry* g, uint32_t occ_mask, uint32_t profile, int32_t* start);

/* Fusion / fission (reading R8) on the partition with occupancy occ_mask and instance starts
 * start_mask (bit i = an instance starts at memory slot i), busy_mask = the slots of busy instances: among the
 * placements of `profile` that overlap at least one instance and no busy slot, the one maximising (fcr of the
 * result, -#destroyed instances, start). *start = its start (-1 = none), *destroyed = the slots of the destroyed
 * instances. Answered from the slot-level tables the simulation kernel uses. Host-only test hook. */
mig_status mig_geometry_fusion(const mig_geometry* g, uint32_t occ_mask, uint32_t start_mask, uint32_t busy_mask,
                               uint32_t profile, int32_t* start, uint32_t* destroyed);

/* ------------------------------------------------------------------------------------------------------------------
 * Traces (job queues). All jobs of a trace arrive at t = 0 (batch).
 * Record format (tracegen/tracegen.h documents the same layout):
 *   jobs[j]     = {x, y, z, w} u32:
 *                 STATIC/MODEL: x = est_mib (compile-time / model-size estimate), y = true_mib (footprint)
 *                 DYNAMIC:      x = b_mib (intercept), y = q0_q16 (inverse reuse ratio at t=0, Q16)
 *                 z = iters (bits 0-15) | class (bits 16-23: 0 STATIC, 1 MODEL, 2 DYNAMIC)
 *                     | PCIe transfer fraction F of an iteration in 1/256 (bits 24-31; MIG_PCIE_CONTENTION)
 *                 w = iter_ticks
 *   jobs_ext[j] = {ws_mib, warps, slope_q8, sigma_mib | qslope_q16 << 16} or NULL (all zero).
 *   Domain: est_mib + ws_mib + ctx_mib is taken modulo 2^32 (u32, as the oracle's req0), and true_mib + ws_mib +
 *   ctx_mib must stay below 2^32 MiB (the kernels saturate it there; the oracle keeps it exact).
 *   DYNAMIC jobs report per-iteration samples (requested MiB, inverse reuse Q16) drawn in-kernel from the
 *   counter-based generator of tracegen.h keyed by (seed, trace_id0 + trace, job index in trace).
 * ---------------------------------------------------------------------------------------------------------------- */
typedef struct {
    const void* jobs;           /* 16 B per job; points at the record of job trace_off[0]                */
    const void* jobs_ext;       /* 16 B per job or NULL                                                  */
    const uint64_t* trace_off;  /* n_traces + 1 CSR offsets (non-decreasing)                             */
    uint64_t n_traces;
    uint64_t trace_id0;         /* global id of trace 0 (sample-generator counter)                       */
    uint64_t seed;              /* sample-generator seed                                                 */
    uint64_t n_jobs;            /* trace_off[n_traces] - trace_off[0] (sizes internal estimate scratch)  */
    uint32_t max_jobs;          /* upper bound on jobs per trace, 1..MIG_MAX_JOBS_PER_TRACE               */
    uint32_t flags;             /* MIG_TRACES_* hints, or 0                                              */
    /* Recorded per-iteration samples (requested MiB and inverse reuse ratio per iteration), or NULL
     * to draw them from the generator. samples points at the sample of index sample_off[0]; DYNAMIC job j's
     * iteration i (1-based) is samples[sample_off[j] - sample_off[0] + i - 1] = {req_mib, inv_reuse_q16}, and
     * sample_off[j+1] - sample_off[j] must be >= its iteration count. sample_off has n_jobs + 1 entries aligned
     * with the job records (jobs[k] <-> sample_off[k]). */
    const void* samples;        /* 8 B per sample (uint2)                                                */
    const uint64_t* sample_off; /* n_jobs + 1, or NULL when samples is NULL                              */
    /* Arrival streams (reading R40; the paper's setting is batch, all at t = 0): arrival
     * tick of every job, aligned with the job records (points at the tick of job trace_off[0]), non-decreasing
     * within a trace (a decrease is flagged MIG_ERR_BAD_RECORD), or NULL = batch. A job joins the queue tail at
     * its arrival, after the requeues of that tick's events; every arrival wakes the scheduler (R9);
     * turnaround = completion - arrival; makespan = the last tick with an end or an arrival. Not with MIG_SCHEME_A
 * (MIG_E_INVALID_ARG). */
    const uint32_t* arrival;
} mig_traces;

#define MIG_MAX_JOBS_PER_TRACE 768 /* on-chip (shared-memory) staging limit of one trace */

/* mig_traces.flags. MIG_TRACES_NO_DYNAMIC: the caller asserts that no job has class DYNAMIC. Only DYNAMIC jobs
 * need the time-series estimator (Alg. 3; the STATIC / MODEL estimate est + ws + ctx, PAPER.md:210,
 * is formed inside the simulation kernels), so mig_simulate then skips the estimator pass over the job records
 * (one HBM read of every record). A DYNAMIC record met under this flag is reported as MIG_ERR_BAD_RECORD in
 * mig_policy_totals.error_flags and simulated without a forecast (no OOM and no early restart for it); its
 * trace's results are then not meaningful. mig_estimate_memory ignores the flag. */
#define MIG_TRACES_NO_DYNAMIC 1u

/* ------------------------------------------------------------------------------------------------------------------
 * Policies
 * ---------------------------------------------------------------------------------------------------------------- */
enum {
    MIG_BASELINE = 0,      /* non-partitioned GPU, one job at a time, queue order       */
    MIG_STATIC = 1,        /* fixed slice layout, no reconfiguration                      */
    MIG_DYNAMIC = 2,       /* create a tight slice on demand (Alg. 2), destroy it at run end               */
    MIG_FUSION_FISSION = 3, /* Scheme B: reuse idle tight slice, Alg. 2, merge/split idle slices, wait     */
    MIG_SCHEME_A = 4        /* Scheme A schedule_by_group: size groups in ascending memory
                               order, each on its homogeneous layout (geometry "scheme_a_layouts"), static
                               round-robin division over the group's slices, reconfiguration when a group drains */
};
enum {
    MIG_EARLY_RESTART = 1, /* preempt when the converged forecast exceeds the slice   */
    MIG_WARP_FOLD = 2,     /* tight fit keeps the full-GPU wave count                        */
    MIG_EWMA_REUSE = 4,    /* EWMA of the inverse reuse ratio instead of its trend (north_star; not in paper) */
    MIG_WAVE_TIME = 8,     /* iter_ticks are full-GPU times; on profile p an iteration of a job with W warps takes
                              ceil(ticks * waves(W,p) / waves(W,full)) ticks (R31 variant)  */
    MIG_PCIE_CONTENTION = 16 /* PCIe bandwidth is divided equally among the runs that transfer (PAPER.md:696-701,
                              reading R39): a run of a job with transfer fraction F/256 (record bits 24-31) > 0
                              advances at 2^24 / (256 - F + F*c) units of 2^-16 nominal ticks per tick while c
                              transferring runs are in progress, re-timed whenever c changes; power, memory
                              integral and waste use actual durations. Lane kernel only (MIG_E_CUDA otherwise). */
};

typedef struct {
    uint32_t kind, flags;
    uint32_t ctx_mib;        /* CUDA context per job                                  */
    uint32_t reconfig_ticks; /* delay before a job starts on a newly created instance                   */
    uint32_t idle_w, w_per_slice;
    double z;                /* z-score of the one-sided 99% bound, default 2.326          */
    uint32_t eps_num, eps_den; /* convergence: |dP| * eps_den < P * eps_num (default 1/100)               */
    uint32_t conv_k;         /* consecutive small changes (default 3, 1..8)                              */
    uint32_t min_n;          /* first iteration with a prediction (default 3, >= 3)                      */
} mig_policy;

/* ------------------------------------------------------------------------------------------------------------------
 * Outputs
 * ---------------------------------------------------------------------------------------------------------------- */
#define MIG_NEVER 0xFFFFu

typedef struct {             /* 80 B, one per job                                                          */
    uint32_t req0_mib;       /* first memory requirement: est + ws + ctx, or the smallest slice (DYNAMIC) */
    uint32_t pred_mib;       /* converged forecast incl. ws + ctx (DYNAMIC), else 0                       */
    uint16_t conv_iter;      /* iteration at which the forecast converged (DYNAMIC), 0 = never            */
    uint16_t n_levels;
    uint16_t fe[6];          /* first iteration whose physical memory exceeds memory level l; MIG_NEVER   */
    double phi, a, sigma;    /* diagnostics of the last fit (DYNAMIC)                                     */
    uint32_t mem_fe[5];      /* sum of the physical MiB over iterations 1..fe[l] (0 if fe[l] = NEVER)     */
    uint32_t mem_conv;       /* ... over iterations 1..conv_iter                                          */
    uint32_t mem_T;          /* ... over all iterations                                                   */
    uint32_t reserved;
} mig_job_estimate;

typedef struct {             /* 96 B, one per (trace, policy)                                             */
    uint32_t makespan, n_jobs, completed, rejected, failed, ooms, preempts, restarts, placements, waits,
        creates, destroys;
    uint64_t energy_wticks, turnaround_sum, busy_slice_ticks, decision_hash;
    uint64_t mem_mib_ticks;  /* integral of the running jobs' physical MiB over time; memory utilisation =
                                mem_mib_ticks / (GPU MiB * makespan)                      */
    uint64_t wasted_ticks;   /* duration of runs that ended in OOM or early restart */
} mig_trace_result;

#define MIG_ERR_TRACE_TOO_LONG 1ull /* a trace has more than max_jobs jobs                             */
#define MIG_ERR_BAD_RECORD 2ull     /* class > 2, iters > 4096, or a sample outside the predictor's range */
#define MIG_ERR_TICK_OVERFLOW 4ull  /* a run's end tick exceeds 2^32 - 1 (ticks are u32; the trace's times wrapped) */

typedef struct {             /* 192 B, one per policy: sums over traces (integer, exact in any order)     */
    uint64_t n_traces, n_jobs, completed, rejected, failed, ooms, preempts, restarts, placements, waits,
        creates, destroys, makespan_sum, makespan_max, energy_wticks, turnaround_sum, busy_slice_ticks,
        decision_hash_sum, mem_mib_ticks, wasted_ticks, error_flags, reserved[3];
} mig_policy_totals;

/* Per-job estimates for every job of the traces (DEVICE buffers; out has trace_off[n]-trace_off[0] entries).
 * stream: a cudaStream_t (NULL = legacy default stream). */
mig_status mig_estimate_memory(const mig_geometry* g, const mig_traces* traces, const mig_policy* policy,
                               mig_job_estimate* out, void* stream);

/* Simulate every trace under each of n_policies policies (host array). Policies must agree on the estimation
 * parameters (ctx_mib, z, eps, conv_k, min_n, EWMA flag). est: per-job estimates from mig_estimate_memory
 * (DEVICE) or NULL (computed internally into stream-ordered scratch). out: DEVICE [n_traces][n_policies] or NULL.
 * totals: DEVICE [n_policies] or NULL; zeroed and accumulated by the call. */
mig_status mig_simulate(const mig_geometry* g, const mig_traces* traces, const mig_policy* policies,
                        uint32_t n_policies, const mig_job_estimate* est, mig_trace_result* out,
                        mig_policy_totals* totals, void* stream);

/* Same as mig_simulate with every pointer of `traces`, `out` and `totals` in HOST memory (page-locked memory
 * recommended). Copies in, estimates, simulates and copies back in chunks pipelined over two streams on the
 * current device; returns after the results are in host memory. out may be NULL: then no per-trace results are
 * written or copied back, only the per-policy totals. */
mig_status mig_simulate_host(const mig_geometry* g, const mig_traces* traces, const mig_policy* policies,
                             uint32_t n_policies, mig_trace_result* out, mig_policy_totals* totals);

/* Workspace of third-party libraries: parse a CUBLAS_WORKSPACE_CONFIG string
 * ":SIZE_KiB:COUNT[,:SIZE_KiB:COUNT...]" (empty = 0) and return sum(SIZE*1024*COUNT) * n_layers bytes in *bytes
 * (SPEC.md:228-236). Host only. MIG_E_PARSE on a malformed string. */
mig_status mig_workspace_bytes(const char* cublas_workspace_config, uint32_t n_layers, uint64_t* bytes);

/* Recorded per-iteration samples of one job (the predictor on recorded traces; the samples
 * Alg. 3 appends each iteration) from a CSV trace file in SPEC.md's format: header
 * `iteration,requested_bytes,reuse_ratio`, one row per iteration, iterations 1, 2, 3, ... in order. Each row becomes
 * one mig_traces sample {req_mib, inv_reuse_q16}: req_mib = ceil(requested_bytes / 2^20) (the requested memory in
 * MiB, R35), inv_reuse_q16 = round(65536 / reuse_ratio) (the inverse reuse ratio in Q16, R22: physical = requested
 * / inverse reuse, so a reuse_ratio in (0, 1] gives inv_reuse >= 1.0). Host only. samples: HOST u32[2 * cap]
 * ({req_mib, inv_reuse_q16} per sample) or NULL to count; *n_out = the number of rows (the samples written when
 * n_out <= cap). MIG_E_IO if the file cannot be read; MIG_E_PARSE (message: line number) on a bad header or row, an
 * iteration out of order, requested_bytes >= 2^52, a reuse_ratio not in (2^-10, 2^10) or a value beyond u32;
 * MIG_E_CAPACITY when samples != NULL and the file has more than cap rows. */
mig_status mig_samples_load_csv(const char* path, uint32_t* samples, uint64_t cap, uint64_t* n_out);

/* Test hook (DEVICE buffers, stream-ordered): out[i] = floor(y[i] * 2^16 / q[i]) computed the way k_estimate maps a
 * requested MiB to physical MiB under inverse reuse q (reading R22) on its fast path: a float estimate corrected
 * by one integer remainder test. Defined for y < 2^18 and 2^16 <= q < 2^26 (the estimator's in-range inputs);
 * other inputs give unspecified values. MIG_E_INVALID_ARG on null pointers with n > 0, MIG_E_CUDA on launch
 * failure. */
mig_status mig_debug_phys_div(const uint32_t* y, const uint32_t* q, uint32_t* out, uint64_t n, void* stream);

/* ------------------------------------------------------------------------------------------------------------------
 * Alg. 1 on the device for larger slot geometries
 * precompute_reachability (PAPER.md:459-474; "can be precomputed offline", :492) for an n_slots-slot GPU,
 * 1 <= n_slots <= 24 (the loaded geometries have <= 8 slots and are tabled on the host). placement_masks: HOST
 * array of the n_placements legal placements (bit i = memory slot i; 1..1024, each non-empty and inside the slots;
 * two profiles may share a mask, e.g. 3g.20gb@0 and 4g.20gb@0). A partition state is a set of disjoint placements;
 * it is final when no placement fits in its free slots (R2); its fcr is the number of distinct final states that
 * adding placements can reach, which depends only on its occupancy (R3). fcr: DEVICE u32[2^n_slots], fcr[m] of
 * every state with occupancy m (0 where no state has occupancy m); state_flags: DEVICE u8[2^n_slots] (bit 0 = some
 * state has occupancy m, bit 1 = final) or NULL; info: HOST, filled when the call returns (it synchronises
 * `stream`) with |S| (states), |F| (finals) and fcr(s0) = |F|. Compute slices are not modelled: in the MIG tables
 * a profile's compute slices lie inside its memory range, so disjoint memory implies disjoint compute (R1).
 * Work: 3^n_slots submask visits. MIG_E_INVALID_ARG on bad sizes or masks, MIG_E_CAPACITY when a count exceeds
 * 2^32 - 1, MIG_E_CUDA on a CUDA failure.
 * ---------------------------------------------------------------------------------------------------------------- */
typedef struct {
    uint64_t n_states, n_finals, fcr_s0;
} mig_reach_info;
mig_status mig_reachability(uint32_t n_slots, const uint32_t* placement_masks, uint32_t n_placements, uint32_t* fcr,
                            uint8_t* state_flags, mig_reach_info* info, void* stream);

/* Number of kernel launches issued by the last device call on this thread (bench accounting). */
uint32_t mig_last_launch_count(void);

/* Device scratch (estimates of DYNAMIC jobs, requeue FIFOs, per-lane partial totals, host-pipeline chunks) comes
 * from a memory pool private to the library, one per device, created on first use; it keeps its memory between
 * calls (large per-call scratch is not re-mapped every call) and never changes the device's default pool.
 * mig_release_scratch returns the unused part of every such pool to the device (call it after the streams that
 * used the library are synchronised). MIG_E_CUDA on failure. */
mig_status mig_release_scratch(void);

/* Kernel timing (bench accounting). While enabled on a thread, every device call of that thread brackets its
 * kernel launches with CUDA events on the call's stream, grouped as "k_estimate" (the estimation kernel),
 * "k_simulate" (all simulation kernels of the call) and, inside it, one group per lane-kernel policy launch
 * ("sim_baseline", "sim_static", "sim_dynamic", "sim_ff", "sim_scheme_a"; a trailing "~" marks a launch on the
 * library's side stream, whose span starts at the fork and includes its wait for SMs: the policy launches of one
 * call alternate between the caller's stream and one forked side stream, joined before the call returns; set
 * MIG_CONCURRENT_POLICIES=0 to serialise them). mig_timing_query synchronises the recorded events,
 * writes up to cap entries {name, total milliseconds, launch count} and clears the record. Enabling or disabling
 * clears it. */
typedef struct {
    char name[16];
    double ms;
    uint32_t launches, reserved;
} mig_kernel_time;
void mig_timing_enable(int on);
mig_status mig_timing_query(mig_kernel_time* out, uint32_t cap, uint32_t* n_out);

#ifdef __cplusplus
}
#endif

#endif /* MIG_H */
