// capi.cu — the extern "C" entry points of libmig.so (include/mig.h): argument validation, per-device geometry
// upload, stream-ordered scratch, kernel launches, and the host-buffer pipeline of mig_simulate_host.
#include <errno.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cmath>

#include <algorithm>
#include <vector>

#include "device_common.cuh"

namespace mig {
cudaError_t launch_estimate(const DevGeom& G, const mig_traces& tr, const mig_policy& pol, mig_job_estimate* out,
                            unsigned long long* scratch, int sm_count, bool dyn_only, cudaStream_t stream);
cudaError_t launch_simulate(const DevGeom* Gdev, const mig_traces& tr, const mig_policy* pols, uint32_t n_pol,
                            const mig_job_estimate* est, mig_trace_result* out, mig_policy_totals* totals,
                            unsigned long long* counter, const unsigned long long* est_err, int sm_count,
                            cudaStream_t stream, uint32_t* launches, uint32_t n_prof, const uint16_t* sid,
                            const uint32_t* a7, uint32_t n_a7, const DevGeom* Gh);
cudaError_t launch_phys_div(const uint32_t* y, const uint32_t* q, uint32_t* out, uint64_t n, cudaStream_t s);
bool simulate_lane_path(uint32_t n_prof, const void* sid, const void* a7);
}  // namespace mig

namespace {
constexpr size_t kCounterBytes = 16 * sizeof(unsigned long long);
thread_local std::string t_err;
thread_local uint32_t t_launches = 0;

// mig_timing_enable / mig_timing_query: events bracketing each group of launches (name, start, stop, launches)
struct TimedRec {
    const char* name;
    cudaEvent_t a, b;
    uint32_t launches;
};
thread_local bool t_timing = false;
thread_local std::vector<TimedRec> t_recs;

void clear_recs() {
    for (auto& r : t_recs) {
        cudaEventDestroy(r.a);
        cudaEventDestroy(r.b);
    }
    t_recs.clear();
}

// Runs launch() (which returns the number of kernels it launched, or -1 on error) between two events when timing.
template <class F>
cudaError_t timed(const char* name, cudaStream_t s, F&& launch) {
    if (!t_timing) return launch(nullptr);
    TimedRec r{name, nullptr, nullptr, 0};
    cudaError_t e = cudaEventCreate(&r.a);
    if (e == cudaSuccess) e = cudaEventCreate(&r.b);
    if (e == cudaSuccess) e = cudaEventRecord(r.a, s);
    if (e != cudaSuccess) return e;
    e = launch(&r.launches);
    if (e == cudaSuccess) e = cudaEventRecord(r.b, s);
    if (e != cudaSuccess) {
        cudaEventDestroy(r.a);
        cudaEventDestroy(r.b);
        return e;
    }
    t_recs.push_back(r);
    return cudaSuccess;
}

mig_status cuda_fail(cudaError_t e, const char* what) {
    return mig_set_error(MIG_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

int sm_count_of(int dev) {
    static int cache[64] = {0};
    if (dev < 0 || dev >= 64) return 148;
    if (!cache[dev]) {
        int n = 0;
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        cache[dev] = n > 0 ? n : 148;
    }
    return cache[dev];
}

// The library's private scratch pool of a device, created on first use (release threshold: keep everything, the
// pool is the library's own; mig_release_scratch trims it).
std::mutex g_pool_mu;
cudaMemPool_t g_pool[64] = {};

cudaError_t scratch_pool(int dev, cudaMemPool_t* out) {
    if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
    std::lock_guard<std::mutex> lock(g_pool_mu);
    if (!g_pool[dev]) {
        cudaMemPoolProps props;
        memset(&props, 0, sizeof(props));
        props.allocType = cudaMemAllocationTypePinned;
        props.handleTypes = cudaMemHandleTypeNone;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = dev;
        cudaMemPool_t p;
        cudaError_t e = cudaMemPoolCreate(&p, &props);
        if (e != cudaSuccess) return e;
        uint64_t thr = ~0ull;
        cudaMemPoolSetAttribute(p, cudaMemPoolAttrReleaseThreshold, &thr);
        g_pool[dev] = p;
    }
    *out = g_pool[dev];
    return cudaSuccess;
}

mig_status device_geometry(const mig_geometry* gc, mig::DevGeom** out, int* dev_out) {
    mig_geometry* g = const_cast<mig_geometry*>(gc);
    int dev = -1;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "no CUDA device (libmig has no CPU fallback)");
    if (dev < 0 || dev >= 64) return mig_set_error(MIG_E_UNSUPPORTED, "device ordinal >= 64");
    std::lock_guard<std::mutex> lock(g->mu);
    if (!g->dev[dev]) {
        mig::DevGeom* p = nullptr;
        e = cudaMalloc(&p, sizeof(mig::DevGeom));
        if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(geometry)");
        e = cudaMemcpy(p, &g->dg, sizeof(mig::DevGeom), cudaMemcpyHostToDevice);
        if (e != cudaSuccess) {
            cudaFree(p);
            return cuda_fail(e, "cudaMemcpy(geometry)");
        }
        g->dev[dev] = p;
    }
    if (!g->sid_dev[dev] && !g->sid16.empty()) {
        uint16_t* t = nullptr;
        const size_t bytes = g->sid16.size() * sizeof(uint16_t);
        e = cudaMalloc(&t, bytes);
        if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(state ids)");
        e = cudaMemcpy(t, g->sid16.data(), bytes, cudaMemcpyHostToDevice);
        if (e != cudaSuccess) {
            cudaFree(t);
            return cuda_fail(e, "cudaMemcpy(state ids)");
        }
        g->sid_dev[dev] = t;
    }
    if (!g->a7_dev[dev] && !g->a7.empty()) {
        uint32_t* t = nullptr;
        const size_t bytes = g->a7.size() * sizeof(uint32_t);
        e = cudaMalloc(&t, bytes);
        if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(fusion/fission table)");
        e = cudaMemcpy(t, g->a7.data(), bytes, cudaMemcpyHostToDevice);
        if (e != cudaSuccess) {
            cudaFree(t);
            return cuda_fail(e, "cudaMemcpy(fusion/fission table)");
        }
        g->a7_dev[dev] = t;
    }
    *out = g->dev[dev];
    *dev_out = dev;
    return MIG_OK;
}

mig_status check_traces(const mig_traces* tr) {
    if (!tr) return mig_set_error(MIG_E_INVALID_ARG, "traces is NULL");
    if (tr->n_traces > 0 && (!tr->jobs || !tr->trace_off))
        return mig_set_error(MIG_E_INVALID_ARG, "traces.jobs and traces.trace_off are required");
    if (tr->max_jobs < 1 || tr->max_jobs > MIG_MAX_JOBS_PER_TRACE)
        return mig_set_error(MIG_E_INVALID_ARG, "traces.max_jobs must be 1.." +
                                                    std::to_string(MIG_MAX_JOBS_PER_TRACE));
    if (tr->flags & ~MIG_TRACES_NO_DYNAMIC) return mig_set_error(MIG_E_INVALID_ARG, "unknown traces.flags bit");
    if ((tr->samples == nullptr) != (tr->sample_off == nullptr))
        return mig_set_error(MIG_E_INVALID_ARG, "traces.samples and traces.sample_off go together");
    return MIG_OK;
}

mig_status check_policy(const mig_policy& p) {
    if (p.kind > MIG_SCHEME_A) return mig_set_error(MIG_E_INVALID_ARG, "policy.kind out of range");
    if (p.flags & ~31u) return mig_set_error(MIG_E_INVALID_ARG, "unknown policy flag");
    if (p.min_n < 3) return mig_set_error(MIG_E_INVALID_ARG, "policy.min_n must be >= 3");
    if (p.conv_k < 1 || p.conv_k > 32) return mig_set_error(MIG_E_INVALID_ARG, "policy.conv_k must be 1..32");
    if (p.eps_den == 0) return mig_set_error(MIG_E_INVALID_ARG, "policy.eps_den must be > 0");
    if (!(p.z >= 0.0 && p.z < 1e6)) return mig_set_error(MIG_E_INVALID_ARG, "policy.z must be in [0, 1e6)");
    return MIG_OK;
}

mig_status check_policies(const mig_geometry* g, const mig_policy* pols, uint32_t n, const mig_traces* tr) {
    if (!pols || n < 1 || n > (uint32_t)mig::kMaxPolicies)
        return mig_set_error(MIG_E_INVALID_ARG, "n_policies must be 1..8");
    for (uint32_t i = 0; i < n; ++i) {
        mig_status s = check_policy(pols[i]);
        if (s != MIG_OK) return s;
        if (tr->arrival && pols[i].kind == MIG_SCHEME_A)
            return mig_set_error(MIG_E_INVALID_ARG, "MIG_SCHEME_A groups the whole queue at t = 0: no arrival streams");
        if (pols[i].kind == MIG_STATIC && g->dg.n_layout == 0)
            return mig_set_error(MIG_E_INVALID_ARG, "MIG_STATIC needs a geometry with a static_layout");
        if (pols[i].kind == MIG_SCHEME_A && !g->info.scheme_a)
            return mig_set_error(MIG_E_INVALID_ARG, "MIG_SCHEME_A needs scheme_a_layouts for every memory level");
        const mig_policy& a = pols[0];
        const mig_policy& b = pols[i];
        if (a.ctx_mib != b.ctx_mib || a.z != b.z || a.eps_num != b.eps_num || a.eps_den != b.eps_den ||
            a.conv_k != b.conv_k || a.min_n != b.min_n || ((a.flags ^ b.flags) & MIG_EWMA_REUSE))
            return mig_set_error(MIG_E_INVALID_ARG, "policies of one mig_simulate call must share ctx_mib, z, eps, "
                                                    "conv_k, min_n and the EWMA flag (one estimate per job)");
    }
    return MIG_OK;
}

// Device path shared by mig_simulate and the host pipeline. counters: kCounterBytes of zeroed scratch
// ([0] estimate, [1] estimate error word, [2..] simulate trace counters).
mig_status simulate_device(const mig_geometry* g, mig::DevGeom* Gdev, int dev, const mig_traces& tr,
                           const mig_policy* pols, uint32_t n_pol, const mig_job_estimate* est,
                           mig_job_estimate* est_scratch, mig_trace_result* out, mig_policy_totals* totals,
                           unsigned long long* counters, cudaStream_t s) {
    cudaError_t e;
    uint32_t launches = 0;
    // MIG_TRACES_NO_DYNAMIC: no estimates are needed (the lane kernels form the STATIC / MODEL estimate themselves
    // and flag a DYNAMIC record); the group kernel always gets them
    const bool skip_est = !est && (tr.flags & MIG_TRACES_NO_DYNAMIC) && mig::simulate_lane_path(g->dg.n_prof,
                                                                                                 g->sid_dev[dev], g->a7_dev[dev]);
    if (!est && !skip_est) {
        e = timed("k_estimate", s, [&](uint32_t* nl) {
            if (nl) *nl = 1;
            return mig::launch_estimate(g->dg, tr, pols[0], est_scratch, counters, sm_count_of(dev), true, s);
        });
        if (e != cudaSuccess) return cuda_fail(e, "k_estimate launch");
        ++launches;
        est = est_scratch;
    }
    uint32_t nl = 0;
    e = timed("k_simulate", s, [&](uint32_t* tl) {
        cudaError_t e2 = mig::launch_simulate(Gdev, tr, pols, n_pol, est, out, totals, counters + 2, counters + 1,
                                              sm_count_of(dev), s, &nl, g->dg.n_prof, g->sid_dev[dev],
                                              g->a7_dev[dev], g->n_a7, &g->dg);
        if (tl) *tl = nl;
        return e2;
    });
    if (e != cudaSuccess) return cuda_fail(e, "k_simulate launch");
    launches += nl;
    t_launches += launches;
    return MIG_OK;
}

}  // namespace

cudaError_t mig_scratch_alloc(void** p, size_t bytes, cudaStream_t s) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    cudaMemPool_t pool;
    if (e == cudaSuccess) e = scratch_pool(dev, &pool);
    if (e == cudaSuccess) e = cudaMallocFromPoolAsync(p, bytes ? bytes : 1, pool, s);
    return e;
}

cudaError_t mig_scratch_free(void* p, cudaStream_t s) { return p ? cudaFreeAsync(p, s) : cudaSuccess; }

mig_status mig_set_error(mig_status s, const std::string& msg) {
    t_err = msg;
    return s;
}

void mig_note_launches(uint32_t n) { t_launches += n; }
void mig_set_launches(uint32_t n) { t_launches = n; }

mig_geometry::~mig_geometry() {
    for (int d = 0; d < 64; ++d)
        if (dev[d]) {
            int cur = 0;
            cudaGetDevice(&cur);
            cudaSetDevice(d);
            cudaFree(dev[d]);
            if (sid_dev[d]) cudaFree(sid_dev[d]);
            if (a7_dev[d]) cudaFree(a7_dev[d]);
            cudaSetDevice(cur);
        }
}

extern "C" {

const char* mig_last_error(void) { return t_err.c_str(); }

mig_status mig_debug_phys_div(const uint32_t* y, const uint32_t* q, uint32_t* out, uint64_t n, void* stream) {
    t_launches = 0;
    if (n && (!y || !q || !out)) return mig_set_error(MIG_E_INVALID_ARG, "mig_debug_phys_div: null buffer");
    const cudaError_t e = mig::launch_phys_div(y, q, out, n, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "mig_debug_phys_div launch");
    t_launches = n ? 1u : 0u;
    return MIG_OK;
}

mig_status mig_workspace_bytes(const char* cfg, uint32_t n_layers, uint64_t* bytes) {
    if (!cfg || !bytes) return mig_set_error(MIG_E_INVALID_ARG, "mig_workspace_bytes: null argument");
    uint64_t total = 0;
    const char* p = cfg;
    while (*p == ' ') ++p;
    while (*p) {
        uint64_t v[2];
        for (int k = 0; k < 2; ++k) {
            if (*p != ':') return mig_set_error(MIG_E_PARSE, std::string("expected ':' at offset ") + std::to_string(p - cfg));
            ++p;
            if (*p < '0' || *p > '9') return mig_set_error(MIG_E_PARSE, std::string("expected a number at offset ") + std::to_string(p - cfg));
            uint64_t x = 0;
            while (*p >= '0' && *p <= '9') {
                x = x * 10 + (uint64_t)(*p - '0');
                if (x > (1ull << 40)) return mig_set_error(MIG_E_PARSE, "value too large");
                ++p;
            }
            v[k] = x;
        }
        total += v[0] * 1024ull * v[1];
        if (*p == ',') {
            ++p;
            if (!*p) return mig_set_error(MIG_E_PARSE, "trailing ','");
        } else if (*p) {
            return mig_set_error(MIG_E_PARSE, std::string("unexpected character at offset ") + std::to_string(p - cfg));
        }
    }
    *bytes = total * n_layers;
    return MIG_OK;
}

uint32_t mig_last_launch_count(void) { return t_launches; }

mig_status mig_samples_load_csv(const char* path, uint32_t* samples, uint64_t cap, uint64_t* n_out) {
    if (!path || !n_out) return mig_set_error(MIG_E_INVALID_ARG, "mig_samples_load_csv: null argument");
    FILE* f = fopen(path, "r");
    if (!f) return mig_set_error(MIG_E_IO, std::string("mig_samples_load_csv: cannot open ") + path);
    char line[512];
    uint64_t n = 0, lineno = 1;
    mig_status st = MIG_OK;
    auto bad = [&](const char* why) {
        st = mig_set_error(MIG_E_PARSE, std::string(path) + ":" + std::to_string(lineno) + ": " + why);
    };
    if (!fgets(line, sizeof(line), f)) {
        bad("empty file (expected the header iteration,requested_bytes,reuse_ratio)");
    } else {
        std::string h(line);
        while (!h.empty() && (h.back() == '\n' || h.back() == '\r' || h.back() == ' ')) h.pop_back();
        if (h != "iteration,requested_bytes,reuse_ratio") bad("header must be iteration,requested_bytes,reuse_ratio");
    }
    while (st == MIG_OK && fgets(line, sizeof(line), f)) {
        ++lineno;
        char* p = line;
        while (*p == ' ' || *p == '\t') ++p;
        if (*p == '\n' || *p == '\r' || *p == 0) continue;  // blank line
        char* e = nullptr;
        errno = 0;
        const unsigned long long it = strtoull(p, &e, 10);
        if (e == p || *e != ',' || errno) { bad("bad iteration"); break; }
        if (it != n + 1) { bad("iterations must be 1, 2, 3, ... in order"); break; }
        p = e + 1;
        const double bytes = strtod(p, &e);
        if (e == p || *e != ',' || !(bytes >= 0.0) || bytes >= 4503599627370496.0) { bad("bad requested_bytes"); break; }
        p = e + 1;
        const double r = strtod(p, &e);
        while (*e == ' ' || *e == '\r' || *e == '\n') ++e;
        if (e == p || *e != 0 || !(r > 1.0 / 1024.0 && r < 1024.0)) { bad("bad reuse_ratio"); break; }
        const double mib = std::ceil(bytes / 1048576.0), q = std::nearbyint(65536.0 / r);
        if (mib > 4294967295.0 || q > 4294967295.0) { bad("value beyond u32"); break; }
        if (samples && n < cap) {
            samples[2 * n] = (uint32_t)mib;
            samples[2 * n + 1] = (uint32_t)q;
        }
        ++n;
    }
    fclose(f);
    if (st != MIG_OK) return st;
    *n_out = n;
    if (samples && n > cap) return mig_set_error(MIG_E_CAPACITY, "mig_samples_load_csv: more rows than cap");
    return MIG_OK;
}

mig_status mig_release_scratch(void) {
    std::lock_guard<std::mutex> lock(g_pool_mu);
    for (int d = 0; d < 64; ++d) {
        if (!g_pool[d]) continue;
        cudaError_t e = cudaMemPoolTrimTo(g_pool[d], 0);
        if (e != cudaSuccess) return cuda_fail(e, "mig_release_scratch");
    }
    return MIG_OK;
}

}  // extern "C"

int mig_timed(const char* name, mig_stream_t stream, const std::function<int(uint32_t*)>& f) {
    return (int)timed(name, (cudaStream_t)stream, [&](uint32_t* nl) { return (cudaError_t)f(nl); });
}

extern "C" {

void mig_timing_enable(int on) {
    clear_recs();
    t_timing = on != 0;
}

mig_status mig_timing_query(mig_kernel_time* out, uint32_t cap, uint32_t* n_out) {
    if (!n_out || (cap && !out)) return mig_set_error(MIG_E_INVALID_ARG, "mig_timing_query: null argument");
    std::vector<mig_kernel_time> agg;
    for (auto& r : t_recs) {
        cudaError_t e = cudaEventSynchronize(r.b);
        float ms = 0.f;
        if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, r.a, r.b);
        if (e != cudaSuccess) {
            clear_recs();
            return cuda_fail(e, "mig_timing_query");
        }
        mig_kernel_time* k = nullptr;
        for (auto& x : agg)
            if (strncmp(x.name, r.name, sizeof(x.name)) == 0) k = &x;
        if (!k) {
            mig_kernel_time z;
            memset(&z, 0, sizeof(z));
            strncpy(z.name, r.name, sizeof(z.name) - 1);
            agg.push_back(z);
            k = &agg.back();
        }
        k->ms += ms;
        k->launches += r.launches;
    }
    clear_recs();
    *n_out = (uint32_t)agg.size();
    for (uint32_t i = 0; i < cap && i < agg.size(); ++i) out[i] = agg[i];
    return MIG_OK;
}

mig_status mig_estimate_memory(const mig_geometry* g, const mig_traces* traces, const mig_policy* policy,
                               mig_job_estimate* out, void* stream) {
    t_launches = 0;
    if (!g || !policy) return mig_set_error(MIG_E_INVALID_ARG, "mig_estimate_memory: null argument");
    mig_status st = check_traces(traces);
    if (st != MIG_OK) return st;
    st = check_policy(*policy);
    if (st != MIG_OK) return st;
    if (traces->n_traces == 0) return MIG_OK;
    if (!out) return mig_set_error(MIG_E_INVALID_ARG, "mig_estimate_memory: out is NULL");
    mig::DevGeom* Gdev;
    int dev;
    st = device_geometry(g, &Gdev, &dev);
    if (st != MIG_OK) return st;
    cudaStream_t s = (cudaStream_t)stream;
    unsigned long long* scratch = nullptr;
    cudaError_t e = mig_scratch_alloc((void**)&scratch, 2 * sizeof(unsigned long long), s);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMallocAsync(scratch)");
    cudaMemsetAsync(scratch, 0, 2 * sizeof(unsigned long long), s);
    e = timed("k_estimate", s, [&](uint32_t* nl) {
        if (nl) *nl = 1;
        return mig::launch_estimate(g->dg, *traces, *policy, out, scratch, sm_count_of(dev), false, s);
    });
    mig_scratch_free(scratch, s);
    if (e != cudaSuccess) return cuda_fail(e, "k_estimate launch");
    t_launches = 1;
    return MIG_OK;
}

mig_status mig_simulate(const mig_geometry* g, const mig_traces* traces, const mig_policy* policies,
                        uint32_t n_policies, const mig_job_estimate* est, mig_trace_result* out,
                        mig_policy_totals* totals, void* stream) {
    t_launches = 0;
    if (!g) return mig_set_error(MIG_E_INVALID_ARG, "mig_simulate: geometry is NULL");
    mig_status st = check_traces(traces);
    if (st != MIG_OK) return st;
    st = check_policies(g, policies, n_policies, traces);
    if (st != MIG_OK) return st;
    cudaStream_t s = (cudaStream_t)stream;
    mig::DevGeom* Gdev;
    int dev;
    st = device_geometry(g, &Gdev, &dev);
    if (st != MIG_OK) return st;
    if (totals) {
        cudaError_t e = cudaMemsetAsync(totals, 0, sizeof(mig_policy_totals) * n_policies, s);
        if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync(totals)");
    }
    if (traces->n_traces == 0) return MIG_OK;
    const bool skip_est = !est && (traces->flags & MIG_TRACES_NO_DYNAMIC) &&
                          mig::simulate_lane_path(g->dg.n_prof, g->sid_dev[dev], g->a7_dev[dev]);
    size_t est_bytes = (est || skip_est) ? 0 : traces->n_jobs * sizeof(mig_job_estimate);
    uint8_t* scratch = nullptr;
    cudaError_t e = mig_scratch_alloc((void**)&scratch, kCounterBytes + est_bytes, s);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMallocAsync(scratch)");
    e = cudaMemsetAsync(scratch, 0, kCounterBytes, s);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync(scratch)");
    st = simulate_device(g, Gdev, dev, *traces, policies, n_policies, est,
                         (est || !est_bytes) ? nullptr : reinterpret_cast<mig_job_estimate*>(scratch + kCounterBytes),
                         out, totals,
                         reinterpret_cast<unsigned long long*>(scratch), s);
    mig_scratch_free(scratch, s);
    return st;
}

mig_status mig_simulate_host(const mig_geometry* g, const mig_traces* traces, const mig_policy* policies,
                             uint32_t n_policies, mig_trace_result* out, mig_policy_totals* totals) {
    t_launches = 0;
    if (!g) return mig_set_error(MIG_E_INVALID_ARG, "mig_simulate_host: geometry is NULL");
    mig_status st = check_traces(traces);
    if (st != MIG_OK) return st;
    st = check_policies(g, policies, n_policies, traces);
    if (st != MIG_OK) return st;
    mig::DevGeom* Gdev;
    int dev;
    st = device_geometry(g, &Gdev, &dev);
    if (st != MIG_OK) return st;
    const mig_traces& T = *traces;
    if (totals) memset(totals, 0, sizeof(mig_policy_totals) * n_policies);
    if (T.n_traces == 0) return MIG_OK;
    // chunking: ~8M jobs (128 MB of records) per chunk, two chunks in flight on two streams. Measured on config 2
    // (1.6 GB of records per call): 2M 36.1 ms, 4M 30.7, 8M 30.6, 16M 31.9 (pipeline fill and drain vs per-chunk
    // overheads); MIG_HOST_CHUNK_JOBS overrides
    uint64_t chunk_jobs = 8ull << 20;
    if (const char* env = getenv("MIG_HOST_CHUNK_JOBS")) chunk_jobs = std::max<uint64_t>(1, strtoull(env, nullptr, 10));
    const uint64_t chunk_traces = std::max<uint64_t>(1, chunk_jobs / T.max_jobs);
    const uint64_t n_chunks = (T.n_traces + chunk_traces - 1) / chunk_traces;
    const uint64_t chunk_jobs_cap = chunk_traces * T.max_jobs;
    auto al = [](size_t x) { return (x + 255) & ~size_t(255); };  // every sub-buffer 256 B aligned
    const size_t jb = al(chunk_jobs_cap * 16), eb = T.jobs_ext ? al(chunk_jobs_cap * 16) : 0,
                 ob = al((chunk_traces + 1) * 8), esb = al(chunk_jobs_cap * sizeof(mig_job_estimate)),
                 rb = al(chunk_traces * n_policies * sizeof(mig_trace_result));
    const size_t ab = T.arrival ? al(chunk_jobs_cap * 4) : 0;  // arrival ticks (R40)
    const size_t per = jb + eb + ob + esb + rb + ab + kCounterBytes;
    cudaStream_t ss[2] = {nullptr, nullptr};
    uint8_t* buf[2] = {nullptr, nullptr};
    std::vector<mig_policy_totals> host_tot(n_chunks * n_policies);
    // per-chunk totals stay on the device until the end (a D2H into pageable memory per chunk would block the
    // host thread and serialise the copy/compute pipeline)
    mig_policy_totals* d_tot_all = nullptr;
    cudaError_t e = cudaMalloc(&d_tot_all, n_chunks * n_policies * sizeof(mig_policy_totals));
    if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(totals)");
    for (int k = 0; k < 2 && st == MIG_OK; ++k) {  // every failure below goes through the one cleanup block
        if ((e = cudaStreamCreateWithFlags(&ss[k], cudaStreamNonBlocking)) != cudaSuccess) {
            ss[k] = nullptr;
            st = cuda_fail(e, "cudaStreamCreate");
        } else if ((e = mig_scratch_alloc((void**)&buf[k], per, ss[k])) != cudaSuccess) {
            buf[k] = nullptr;
            st = cuda_fail(e, "host pipeline scratch");
        }
    }
    const uint64_t* off = T.trace_off;
    for (uint64_t c = 0; c < n_chunks && st == MIG_OK; ++c) {
        const int k = (int)(c & 1);
        cudaStream_t s = ss[k];
        uint8_t* b = buf[k];
        const uint64_t t0 = c * chunk_traces, t1 = std::min<uint64_t>(T.n_traces, t0 + chunk_traces);
        const uint64_t nt = t1 - t0, jlo = off[t0] - off[0], jhi = off[t1] - off[0], nj = jhi - jlo;
        if (nj > chunk_jobs_cap) {
            st = mig_set_error(MIG_E_INVALID_ARG, "a trace exceeds max_jobs");
            break;
        }
        uint8_t* d_jobs = b;
        uint8_t* d_ext = b + jb;
        uint64_t* d_off = reinterpret_cast<uint64_t*>(b + jb + eb);
        mig_job_estimate* d_est = reinterpret_cast<mig_job_estimate*>(b + jb + eb + ob);
        mig_trace_result* d_out = reinterpret_cast<mig_trace_result*>(b + jb + eb + ob + esb);
        mig_policy_totals* d_tot = d_tot_all + c * n_policies;
        uint32_t* d_arr = reinterpret_cast<uint32_t*>(b + jb + eb + ob + esb + rb);
        unsigned long long* d_cnt = reinterpret_cast<unsigned long long*>(b + jb + eb + ob + esb + rb + ab);
        e = cudaMemcpyAsync(d_jobs, (const uint8_t*)T.jobs + jlo * 16, nj * 16, cudaMemcpyHostToDevice, s);
        if (e == cudaSuccess && T.jobs_ext)
            e = cudaMemcpyAsync(d_ext, (const uint8_t*)T.jobs_ext + jlo * 16, nj * 16, cudaMemcpyHostToDevice, s);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(d_off, off + t0, (nt + 1) * 8, cudaMemcpyHostToDevice, s);
        if (e == cudaSuccess && T.arrival)
            e = cudaMemcpyAsync(d_arr, T.arrival + jlo, nj * 4, cudaMemcpyHostToDevice, s);
        uint8_t* d_smp = nullptr;
        uint64_t* d_soff = nullptr;
        if (e == cudaSuccess && T.samples) {  // recorded samples of this chunk's jobs (stream-ordered scratch)
            const uint64_t* so = T.sample_off;
            const uint64_t slo = so[jlo] - so[0], shi = so[jhi] - so[0];
            e = mig_scratch_alloc((void**)&d_smp, (shi - slo) * 8 + 8, s);
            if (e == cudaSuccess) e = mig_scratch_alloc((void**)&d_soff, (nj + 1) * 8, s);
            if (e == cudaSuccess)
                e = cudaMemcpyAsync(d_smp, (const uint8_t*)T.samples + slo * 8, (shi - slo) * 8, cudaMemcpyHostToDevice, s);
            if (e == cudaSuccess) e = cudaMemcpyAsync(d_soff, so + jlo, (nj + 1) * 8, cudaMemcpyHostToDevice, s);
        }
        if (e == cudaSuccess) e = cudaMemsetAsync(d_cnt, 0, kCounterBytes, s);
        if (e == cudaSuccess) e = cudaMemsetAsync(d_tot, 0, n_policies * sizeof(mig_policy_totals), s);
        if (e != cudaSuccess) {
            st = cuda_fail(e, "host pipeline H2D");
            break;
        }
        mig_traces ct = T;
        ct.jobs = d_jobs;
        ct.jobs_ext = T.jobs_ext ? d_ext : nullptr;
        ct.trace_off = d_off;
        ct.n_traces = nt;
        ct.trace_id0 = T.trace_id0 + t0;
        ct.n_jobs = nj;
        ct.samples = d_smp;
        ct.sample_off = d_soff;
        ct.arrival = T.arrival ? d_arr : nullptr;
        st = simulate_device(g, Gdev, dev, ct, policies, n_policies, nullptr, d_est, out ? d_out : nullptr, d_tot, d_cnt,
                             s);  // no per-trace results wanted: none are written
        if (d_smp) mig_scratch_free(d_smp, s);
        if (d_soff) mig_scratch_free(d_soff, s);
        if (st != MIG_OK) break;
        if (out)
            e = cudaMemcpyAsync(out + t0 * n_policies, d_out, nt * n_policies * sizeof(mig_trace_result),
                                cudaMemcpyDeviceToHost, s);
        if (e != cudaSuccess) st = cuda_fail(e, "host pipeline D2H");
    }
    for (int k = 0; k < 2; ++k) {  // cleanup (every path): scratch, streams; the totals buffer below
        if (!ss[k]) continue;
        if (buf[k]) mig_scratch_free(buf[k], ss[k]);
        e = cudaStreamSynchronize(ss[k]);
        if (e != cudaSuccess && st == MIG_OK) st = cuda_fail(e, "host pipeline");
        cudaStreamDestroy(ss[k]);
    }
    if (st == MIG_OK) {
        e = cudaMemcpy(host_tot.data(), d_tot_all, n_chunks * n_policies * sizeof(mig_policy_totals),
                       cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) st = cuda_fail(e, "host pipeline totals D2H");
    }
    cudaFree(d_tot_all);
    if (st != MIG_OK) return st;
    if (totals) {
        for (uint64_t c = 0; c < n_chunks; ++c)
            for (uint32_t p = 0; p < n_policies; ++p) {
                const uint64_t* src = reinterpret_cast<const uint64_t*>(&host_tot[c * n_policies + p]);
                uint64_t* dst = reinterpret_cast<uint64_t*>(&totals[p]);
                for (int f = 0; f < 21; ++f) {
                    if (f == 13) dst[f] = std::max(dst[f], src[f]);
                    else if (f == 20) dst[f] |= src[f];
                    else dst[f] += src[f];
                }
            }
    }
    return MIG_OK;
}

}  // extern "C"
