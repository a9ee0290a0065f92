// estimate.cu — k_estimate: per-job memory estimation.
//
//   STATIC / MODEL jobs: req0 = estimate + workspace + context (compile-time analysis PAPER.md:210, model-size
//   estimation PAPER.md:214, :569; context PAPER.md:345-346; workspace PAPER.md:358-362). The true footprint
//   exceeds a memory level l at iteration 1 or never (R12).
//   DYNAMIC jobs: Alg. 3 PeakMemoryPrediction over the per-iteration samples, plus the
//   first-exceed iteration of every memory level (where the job would OOM).
//
// Layout: one warp per batch of traces (persistent CTAs, atomic counter). Lanes take the jobs 32 at a time;
// each DYNAMIC job is then processed by the whole warp, lanes over iterations: lane i draws sample base+i+1
// in-kernel (counter-based generator, tracegen.h), the exact integer moments Sum y, Sum t*y, Sum y^2, Sum q,
// Sum t*q are warp inclusive scans (__shfl_up_sync), every lane evaluates the forecast P_n for its own n, the
// convergence rule becomes a run of conv_k set bits in a 64-bit window of two __ballot_sync masks, and each
// level's first exceed is one __ballot_sync + __ffs. Arithmetic follows DESIGN.md "Canonical arithmetic"
// (exact int64/int128 moments, one fixed sequence of IEEE double operations, no FMA contraction).
#include "device_common.cuh"
#include "../../tracegen/tracegen.h"  // input generator only: the samples a dynamic job reports

namespace mig {

struct EstParams {
    const uint4* jobs;
    const uint4* ext;
    const uint64_t* off;
    uint64_t n_traces, trace_id0, seed;
    mig_job_estimate* out;
    const uint2* samples;       // recorded samples or NULL (generator)
    const uint64_t* sample_off;
    unsigned long long* counter;
    unsigned long long* err;
    uint32_t ctx, eps_num, eps_den, conv_k, min_n;
    uint32_t dyn_only;  // skip writing STATIC/MODEL estimates (mig_simulate recomputes them while staging)
    uint32_t ewma;      // MIG_EWMA_REUSE (R36): EWMA of the inverse reuse ratio instead of its linear trend
    double z;
};

struct FitOut {
    int64_t P;
    double phi, a, sigma;
};

// One fit + forecast at n samples (oracle: fit_and_predict). The slope
// diagnostic a = 6K/D is computed once for the reported lane (estimate_dynamic). q_unit: the inverse reuse is
// exactly 1.0 at every sample, so its forecast is exactly 65536 and V = 1 (the canonical sequence gives the same).
__device__ __forceinline__ FitOut fit_at(int64_t n, int64_t Sy, int64_t Sty, int64_t Syy, int64_t Sq, int64_t Stq,
                                         int64_t T, double z, int64_t ws_ctx, bool q_unit, bool ewma, int64_t L,
                                         bool small, bool n32) {
    const int64_t n2m1 = n * n - 1;
    const int64_t D = n * n2m1;
    const int64_t Ky = 2 * Sty - (n + 1) * Sy;
    const int64_t h = 2 * T - n - 1;
    // small (y < 2^18, T <= 4096): |Sy (n^2-1)| < 2^54 and |3 Ky h| < 2^57, so numY is exact in int64 and its
    // conversion is the same single rounding as i128_to_double's
    const __int128 numY = small ? (__int128)0 : (__int128)Sy * n2m1 + (__int128)3 * Ky * h;
    const int64_t numY64 = small ? Sy * n2m1 + 3 * Ky * h : 0;
    // n32 (small and n <= 32): Sy < 2^23, Syy < 2^41, |Ky| < 2^29, so every term of the residual sum is below 2^60 and
    // it is exact in int64 (its conversion is the same single rounding as i128_to_double's)
    const __int128 ssrN =
        n32 ? (__int128)0 : (__int128)n2m1 * (__int128)(n * Syy - Sy * Sy) - (__int128)3 * Ky * Ky;  // n*Syy, Sy^2 < 2^62
    const int64_t ssr64 = n32 ? n2m1 * (n * Syy - Sy * Sy) - 3 * Ky * Ky : 0;
    const double den = __ll2double_rn(D);
    FitOut f;
    const double yT = __ddiv_rn(small ? __ll2double_rn(numY64) : i128_to_double(numY), den);
    const double var = __ddiv_rn(n32 ? __ll2double_rn(ssr64) : i128_to_double(ssrN), __ll2double_rn(D * (n - 2)));
    f.sigma = __dsqrt_rn(var);
    double u = __dadd_rn(yT, __dmul_rn(z, f.sigma));
    if (u < 0.0) u = 0.0;
    double V = 1.0;
    if (ewma) {  // R36: V = max(L_n / 65536, 1)
        V = __dmul_rn(__ll2double_rn(L), 1.0 / 65536.0);
        if (V < 1.0) V = 1.0;
    } else if (!q_unit) {
        const int64_t Kq = 2 * Stq - (n + 1) * Sq;
        const __int128 numQ = (__int128)Sq * n2m1 + (__int128)3 * Kq * h;
        V = __dmul_rn(__ddiv_rn(i128_to_double(numQ), den), 1.0 / 65536.0);  // exact power-of-two scaling
        if (V < 1.0) V = 1.0;
    }
    // V = 1 exactly for a constant inverse reuse (no EWMA): the IEEE quotient u / 1 is u, so the division is skipped
    f.phi = (q_unit && !ewma) ? u : __ddiv_rn(u, V);
    f.a = 0.0;
    f.P = (int64_t)ceil(f.phi) + ws_ctx;
    return f;
}

__device__ __forceinline__ double slope_of(int64_t n, int64_t Sy, int64_t Sty) {
    const int64_t Ky = 2 * Sty - (n + 1) * Sy;
    return __ddiv_rn(__ll2double_rn(6 * Ky), __ll2double_rn(n * (n * n - 1)));
}

__device__ __forceinline__ void store_estimate(mig_job_estimate* dst, uint32_t req0, uint32_t pred, uint32_t conv,
                                               uint32_t n_levels, const uint32_t fe[5], double phi, double a,
                                               double sigma, const uint32_t mfe[5], uint32_t mconv, uint32_t mT) {
    uint4 w0 = make_uint4(req0, pred, (conv & 0xFFFFu) | (n_levels << 16), fe[0] | (fe[1] << 16));
    uint4 w1 = make_uint4(fe[2] | (fe[3] << 16), fe[4] | (kNever << 16), __double2loint(phi), __double2hiint(phi));
    uint4 w2 = make_uint4(__double2loint(a), __double2hiint(a), __double2loint(sigma), __double2hiint(sigma));
    uint4 w3 = make_uint4(mfe[0], mfe[1], mfe[2], mfe[3]);
    uint4 w4 = make_uint4(mfe[4], mconv, mT, 0u);
    uint4* d = reinterpret_cast<uint4*>(dst);
    d[0] = w0;
    d[1] = w1;
    d[2] = w2;
    d[3] = w3;
    d[4] = w4;
}

// Warp inclusive prefix sum (32-bit).
__device__ __forceinline__ uint32_t warp_scan_u32(uint32_t v, uint32_t lane) {
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t o = __shfl_up_sync(FULL, v, d);
        if (lane >= (uint32_t)d) v += o;
    }
    return v;
}

// floor(y * 2^16 / q), the physical MiB of a requested y under inverse reuse q (R22), for y < 2^18 and
// 2^16 <= q < 2^26 (the quotient is below 2^18). A float estimate (exact y, q rounded to 24 bits, approximate
// reciprocal: relative error below 2^-21, so within 1/8 of the quotient) is off by at most one, and one integer
// remainder test on each side makes it exact. Pinned against integer division on the GPU
// (tests/test_parity_gpu.py::test_exact_division_hook via mig_debug_phys_div).
__device__ __forceinline__ uint32_t phys_div(uint32_t y, uint32_t q) {
    const uint32_t k = __float2uint_rz(__fmul_rn(__uint2float_rn(y), __fdividef(65536.0f, __uint2float_rn(q))));
    const int64_t r = (int64_t)((uint64_t)y << 16) - (int64_t)((uint64_t)k * q);
    return r < 0 ? k - 1u : (r >= (int64_t)q ? k + 1u : k);
}

__global__ void k_phys_div(const uint32_t* y, const uint32_t* q, uint32_t* out, uint64_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = phys_div(y[i], q[i]);
}

cudaError_t launch_phys_div(const uint32_t* y, const uint32_t* q, uint32_t* out, uint64_t n, cudaStream_t s) {
    if (n) k_phys_div<<<1184, 256, 0, s>>>(y, q, out, n);
    return cudaGetLastError();
}

// Samples after the forecast has converged (or when the job is too short to forecast): only the first exceed of
// each memory level and the memory integral remain, so the loop is the sample draw, one level
// ballot per chunk while a level is still reachable, and one reduction. CHECK: per-sample input checks (the range
// bounds could break them, or q may fall below 1.0); QUNIT: constant inverse reuse 1.0 (physical = requested + ws
// + ctx). Without CHECK the inputs satisfy y < 2^18 and 2^16 <= q < 2^26: floor(y * 2^16 / q) by phys_div.
template <bool CHECK, bool QUNIT, bool W32>
__device__ __forceinline__ void scan_tail(const DevGeom& G, const uint2* rec_samples, uint32_t rec_count, uint32_t base,
                                          uint32_t T, uint32_t lane, uint64_t key, uint32_t b, uint32_t slope,
                                          uint32_t sigma_n, uint32_t q0, uint32_t qs, int64_t ws_ctx,
                                          uint64_t phys_hi, uint32_t& lnext, uint32_t& Smem, bool& bad,
                                          uint32_t (&fe)[5], uint32_t (&mfe)[5]) {
    // levels that no sample can exceed are never tested (phys_hi bounds every physical MiB of the job)
    uint32_t lend = lnext;
    while (lend < G.n_levels && G.level_mem[lend] < phys_hi) ++lend;
    uint64_t lvl = lnext < lend ? G.level_mem[lnext] : ~0ull;  // the level being watched (lnext)
    // W32 (no checks, ws + ctx < 2^31): every physical MiB is below 2^32, so the sums and tests run in 32 bits
    const uint32_t wc32 = (uint32_t)ws_ctx;
    uint32_t n = base + lane + 1;  // this lane's iteration (carried, so the lane id is not re-read per chunk)
    auto chunk = [&](bool last) {
        const bool valid = !last || n <= T;
        uint32_t y = 0, q = 0;
        if (valid) {
            if (rec_samples) {
                const uint2 v = __ldg(rec_samples + (n <= rec_count ? n : rec_count) - 1);
                y = v.x;
                q = v.y;
            } else if (CHECK) {
                tg_dyn_sample(key, n, b, slope, sigma_n, q0, qs, &y, &q);
            } else {  // the series' bounds keep the draw in 32-bit range (y_hi < 2^18)
                tg_dyn_sample_fast(key, n, b, slope, sigma_n, q0, qs, &y, &q);
            }
            if (CHECK) bad |= (q == 0) | (y >= (1u << 18)) | (q >= (1u << 26));
        }
        uint64_t phys64 = 0;
        uint32_t phys = 0;
        if (W32) {
            phys = valid ? (QUNIT ? y : phys_div(y, q)) + wc32 : 0u;
            phys64 = phys;
        } else {
            if (valid) {
                if (QUNIT) phys64 = (uint64_t)y + ws_ctx;
                else if (CHECK) phys64 = (q ? ((uint64_t)y * 65536ull) / q : 0ull) + ws_ctx;
                else phys64 = (uint64_t)phys_div(y, q) + ws_ctx;
            }
            phys = (uint32_t)phys64;
        }
        while (lnext < lend) {
            const bool over = W32 ? (valid && phys > (uint32_t)lvl) : (valid && phys64 > lvl);
            const uint32_t m = __ballot_sync(FULL, over);
            if (!m) break;
            const uint32_t src = (uint32_t)__ffs(m) - 1u;
            // the lane id read here, on the (rare) crossing path, not kept live through the chunk loop
            uint32_t lid;
            asm volatile("mov.u32 %0, %%laneid;" : "=r"(lid));
            const uint32_t pre = Smem + __reduce_add_sync(FULL, lid <= src ? phys : 0u);
#pragma unroll
            for (int k = 0; k < kMaxLevels; ++k)
                if ((uint32_t)k == lnext) {
                    fe[k] = base + src + 1u;
                    mfe[k] = pre;
                }
            ++lnext;
            lvl = lnext < lend ? G.level_mem[lnext] : ~0ull;
        }
        Smem += __reduce_add_sync(FULL, phys);
    };
    // full chunks need no per-lane bound test; the last (partial) chunk does
    for (; base + 32 <= T; base += 32, n += 32) chunk(false);
    if (base < T) chunk(true);
}

// Whole-warp estimation of one DYNAMIC job (lanes over iterations).
// PLAIN: generated samples and no EWMA variant (the common case), so those paths compile out.
// A bound on every physical MiB of a DYNAMIC job's generated series, or ~0 when the series' range bounds do not
// keep it inside the predictor's input limits (y < 2^18, 0 < q < 2^26: the checked path). y <= b + slope*T/256 + the
// largest Irwin-Hall draw + 1, q grows from q0 by qs (the draw is at most 510 * sigma * 7094 / 2^20; 131070 / 2^28 =
// 511.99 / 2^20 bounds it); the inverse reuse only grows, so q >= q0, and the division by q0 is bounded from above
// by a shift by floor(log2 q0) (no 64-bit division).
__device__ __forceinline__ uint64_t generated_phys_hi(uint4 r, uint4 e, uint32_t ctx) {
    const uint32_t T = r.z & 0xFFFFu;
    const uint32_t b = r.x, q0 = r.y, slope = e.z, sigma_n = e.w & 0xFFFFu, qs = e.w >> 16;
    const uint64_t y_hi = (uint64_t)b + (((uint64_t)slope * T) >> 8) +
                          (((uint64_t)131070u * ((sigma_n & 0xFFFFu) * 7094u)) >> 28) + 2u;
    const bool check = y_hi >= (1u << 18) || q0 == 0 || (uint64_t)q0 + (uint64_t)qs * T >= (1u << 26);
    const bool q_unit = q0 == 65536u && qs == 0;
    return check ? ~0ull : (q_unit ? y_hi : (y_hi << 16) >> (31 - __clz(q0))) + (uint64_t)e.x + ctx;
}

// key: the job's sample-generator key (tracegen.h tg_job_key, formed for the chunk's jobs in parallel).
template <bool PLAIN>
__device__ __forceinline__ void estimate_dynamic(const DevGeom& G, const EstParams& P, uint64_t key, uint4 r,
                                 uint4 e, uint32_t lane, mig_job_estimate* dst, const uint2* rec_samples,
                                 uint32_t rec_count) {
    if (PLAIN) rec_samples = nullptr;
    const bool ewma = !PLAIN && P.ewma != 0;
    const uint32_t T = r.z & 0xFFFFu;
    const uint32_t b = r.x, q0 = r.y, ws = e.x, slope = e.z, sigma_n = e.w & 0xFFFFu, qs = e.w >> 16;
    const int64_t ws_ctx = (int64_t)ws + P.ctx;
    uint32_t fe[5] = {kNever, kNever, kNever, kNever, kNever};
    uint32_t mfe[5] = {0u, 0u, 0u, 0u, 0u};  // physical MiB summed over iterations 1..fe[l]
    uint32_t Smem = 0, mconv = 0;            // running sum (memory integral)
    auto fe_set = [&](uint32_t l, uint32_t v, uint32_t m) {
#pragma unroll
        for (int k = 0; k < kMaxLevels; ++k)
            if ((uint32_t)k == l) {
                fe[k] = v;
                mfe[k] = m;
            }
    };
    const bool q_unit = !rec_samples && q0 == 65536u && qs == 0;  // generated, constant inverse reuse 1.0
    uint32_t lnext = 0;                          // lowest level whose first exceed is not yet known
    int64_t Sy = 0, Sty = 0, Syy = 0, Sq = 0, Stq = 0, Plast = 0, Lcarry = 0;
    uint32_t okprev = 0, conv = 0, pred = 0;
    double phi = 0.0, a = 0.0, sig = 0.0;
    bool done_pred = T < P.min_n;
    bool bad = false;
    // generated series whose range bounds already satisfy the predictor's input limits skip the per-sample checks;
    // phys_hi bounds every physical MiB of the job
    const uint64_t phys_hi_gen = generated_phys_hi(r, e, P.ctx);  // (formed here: a passed-in copy spills)
    const bool check = rec_samples || phys_hi_gen == ~0ull;
    const bool fastq = !check && q0 >= 65536u;  // phys_div's range: generated q never decreases from q0
    const uint64_t phys_hi = rec_samples ? ~0ull : phys_hi_gen;
    uint32_t base = 0;
    for (; base < T && !done_pred; base += 32) {  // until convergence; then scan_tail to T (memory integral)
        const uint32_t n = base + lane + 1;
        const bool valid = n <= T;
        uint32_t y = 0, q = 0;
        if (valid) {
            if (rec_samples) {  // recorded series (coalesced 8 B loads)
                const uint2 v = __ldg(rec_samples + (n <= rec_count ? n : rec_count) - 1);  // short series: flagged
                y = v.x;
                q = v.y;
            } else if (check) {
                tg_dyn_sample(key, n, b, slope, sigma_n, q0, qs, &y, &q);
            } else {  // the series' bounds keep the draw in 32-bit range (y_hi < 2^18)
                tg_dyn_sample_fast(key, n, b, slope, sigma_n, q0, qs, &y, &q);
            }
            if (check) bad |= (q == 0) | (y >= (1u << 18)) | (q >= (1u << 26));
        }
        // physical MiB of iteration n and its running sum (R22: requested / inverse reuse, + ws + ctx)
        const uint64_t phys64 =
            valid ? (q_unit ? (uint64_t)y : fastq ? phys_div(y, q) : ((uint64_t)y * 65536ull) / q) + ws_ctx : 0ull;
        const uint32_t phys = (uint32_t)phys64;
        // running sum of the memory integral: one reduction per chunk, prefixes only where needed
        auto prefix = [&](uint32_t m) { return Smem + __reduce_add_sync(FULL, lane <= m ? phys : 0u); };
        // first-exceed iteration of every memory level (R12): phys(i) = floor(y*65536/q) + ws + ctx > L.
        // Levels ascend, so fe[l] <= fe[l+1]: only the lowest level not yet crossed needs a ballot per chunk
        // (more when one chunk crosses several levels).
        while (lnext < G.n_levels) {
            const bool over = valid && phys64 > G.level_mem[lnext];
            const uint32_t m = __ballot_sync(FULL, over);
            if (!m) break;
            fe_set(lnext, base + __ffs(m), prefix((uint32_t)__ffs(m) - 1u));
            ++lnext;
        }
        const uint32_t Snext = Smem + __reduce_add_sync(FULL, phys);
        // exact integer moments at n = base + lane + 1 (inclusive warp scans + carried totals)
        const int64_t yi = y, qi = q, ni = n;
        const int64_t sy = Sy + (int64_t)warp_scan_u32(y, lane);  // sum y <= 4096 * 2^18 fits 32 bits
        // first chunk of an in-range series: n*y < 2^23 and the prefix sums stay below 2^28, so the scan runs in 32 bits
        const int64_t sty = (base == 0 && !check) ? (int64_t)warp_scan_u32(valid ? n * y : 0u, lane)
                                                  : Sty + warp_scan_i64(valid ? ni * yi : 0, lane);
        const int64_t syy = Syy + warp_scan_i64(yi * yi, lane);
        // constant inverse reuse: its fit is not needed (V = 1), so its moments are not formed
        const int64_t sq = q_unit ? 0 : Sq + warp_scan_i64(qi, lane);
        const int64_t stq = q_unit ? 0 : Stq + warp_scan_i64(valid ? ni * qi : 0, lane);
        // EWMA of the inverse reuse ratio (R36): L_1 = q_1, L_i = L_{i-1} + ((q_i - L_{i-1}) >> 3); a sequential
        // recurrence, evaluated over the chunk's lanes in order (optional variant, never on the default path).
        int64_t myL = 0;
        if (ewma) {
            int64_t L = Lcarry;
            for (uint32_t k = 0; k < 32; ++k) {
                const int64_t qk = (int64_t)__shfl_sync(FULL, q, k);
                L = (base + k == 0) ? qk : L + ((qk - L) >> 3);
                if (lane == k) myL = L;
            }
            Lcarry = L;
        }
        const bool has = valid && n >= P.min_n;
        FitOut f = {0, 0.0, 0.0, 0.0};
        if (has)
            f = fit_at(ni, sy, sty, syy, sq, stq, T, P.z, ws_ctx, q_unit, ewma, myL, !check && T <= 4096,
                       !check && T <= 4096 && base == 0);
        int64_t Pprev = __shfl_up_sync(FULL, f.P, 1);
        if (lane == 0) Pprev = Plast;
        const bool prev_has = n >= P.min_n + 1;
        const int64_t diff = f.P > Pprev ? f.P - Pprev : Pprev - f.P;
        const bool ok = has && prev_has && (int64_t)P.eps_den * diff < (int64_t)P.eps_num * Pprev;
        const uint32_t M = __ballot_sync(FULL, ok);
        // converged at n <=> the last conv_k relative changes (n-conv_k+1 .. n) were all small (R24)
        const uint64_t X = ((uint64_t)M << 32) | okprev;
        uint64_t Y = X;
        for (uint32_t d = 1; d < P.conv_k; ++d) Y &= X << d;
        const uint32_t cm = (uint32_t)(Y >> 32);
        const uint32_t last_lane = (T - 1 - base) < 32 ? (T - 1 - base) : 31;
        const uint32_t src = cm ? (uint32_t)(__ffs(cm) - 1) : last_lane;
        const int64_t Ps = __shfl_sync(FULL, f.P, src);
        const double phs = __shfl_sync(FULL, f.phi, src), ss = __shfl_sync(FULL, f.sigma, src);
        const int64_t nsrc = base + src + 1, sy_s = __shfl_sync(FULL, sy, src), sty_s = __shfl_sync(FULL, sty, src);
        const double as = (cm || (base + 32 >= T && T >= P.min_n)) ? slope_of(nsrc, sy_s, sty_s) : 0.0;
        if (cm) {
            conv = base + src + 1;
            mconv = prefix(src);
            pred = (uint32_t)Ps;
            phi = phs;
            a = as;
            sig = ss;
            done_pred = true;
        } else {
            if (base + 32 >= T && T >= P.min_n) {  // last chunk, never converged: diagnostics of the fit at n = T
                phi = phs;
                a = as;
                sig = ss;
            }
            Sy = __shfl_sync(FULL, sy, 31);
            Sty = __shfl_sync(FULL, sty, 31);
            Syy = __shfl_sync(FULL, syy, 31);
            Sq = __shfl_sync(FULL, sq, 31);
            Stq = __shfl_sync(FULL, stq, 31);
            Plast = __shfl_sync(FULL, f.P, 31);
            okprev = M;
        }
        Smem = Snext;
    }
    // W32: every physical MiB of the tail is below 2^32 (generated in-range series, ws + ctx < 2^31)
    const bool w32 = !check && ws_ctx < (1ll << 31);
    if (q_unit) {
        if (check) scan_tail<true, true, false>(G, rec_samples, rec_count, base, T, lane, key, b, slope, sigma_n, q0,
                                                qs, ws_ctx, phys_hi, lnext, Smem, bad, fe, mfe);
        else if (w32) scan_tail<false, true, true>(G, rec_samples, rec_count, base, T, lane, key, b, slope, sigma_n,
                                                   q0, qs, ws_ctx, phys_hi, lnext, Smem, bad, fe, mfe);
        else scan_tail<false, true, false>(G, rec_samples, rec_count, base, T, lane, key, b, slope, sigma_n, q0, qs,
                                           ws_ctx, phys_hi, lnext, Smem, bad, fe, mfe);
    } else {  // (q0 < 1.0 takes the checked path: its per-sample checks never fire, its division is exact for any q)
        if (fastq && w32) scan_tail<false, false, true>(G, rec_samples, rec_count, base, T, lane, key, b, slope,
                                                        sigma_n, q0, qs, ws_ctx, phys_hi, lnext, Smem, bad, fe, mfe);
        else if (fastq) scan_tail<false, false, false>(G, rec_samples, rec_count, base, T, lane, key, b, slope,
                                                       sigma_n, q0, qs, ws_ctx, phys_hi, lnext, Smem, bad, fe, mfe);
        else scan_tail<true, false, false>(G, rec_samples, rec_count, base, T, lane, key, b, slope, sigma_n, q0, qs,
                                           ws_ctx, phys_hi, lnext, Smem, bad, fe, mfe);
    }
    if (__any_sync(FULL, bad) && lane == 0) atomicOr(P.err, (unsigned long long)MIG_ERR_BAD_RECORD);
    if (lane == 0) store_estimate(dst, G.mem[0], pred, conv, G.n_levels, fe, phi, a, sig, mfe, mconv, Smem);
}

// Traces are taken kBatch at a time (one atomic per batch); the warp streams the batch's job records as one
// contiguous range, 32 coalesced 16-B records per step, so STATIC/MODEL-only workloads run at scan speed; a DYNAMIC
// job's trace is found by a ballot over the batch's offsets held one per lane.
constexpr uint32_t kEstBatch = 32;

// 5 CTAs x 8 warps per SM (48 registers, 84 B of spills): measured against 3 / 4 / 6 CTAs (80 / 64 / 40 registers),
// config 3 / 4 / 5 k_estimate 11.46 / 85.8 / 162.0 ms at 3 CTAs, 10.75 / 82.1 / 152.9 at 4, 10.72 / 81.5 / 150.3 at
// 5, 10.81 / 81.1 / 149.6 at 6: the per-sample loop is latency-bound (RNG chain, ballots, reductions), so more
// resident warps beat a few spilled registers
#ifndef EST_MINB
#define EST_MINB 5
#endif
template <bool PLAIN>
__global__ void __launch_bounds__(256, EST_MINB) k_estimate(const DevGeom G, const EstParams P) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t j_base = P.off[0];
    __shared__ uint64_t s_tkey[8][32];
    __shared__ uint64_t s_jkey[8][32];  // the generator key of each of the chunk's jobs
    for (;;) {
        unsigned long long t0 = 0;
        if (lane == 0) t0 = atomicAdd(P.counter, (unsigned long long)kEstBatch);
        t0 = __shfl_sync(FULL, t0, 0);
        if (t0 >= P.n_traces) break;
        const uint32_t nb = (uint32_t)min((unsigned long long)kEstBatch, P.n_traces - t0);
        const uint64_t my_off = lane < nb ? P.off[t0 + lane] - j_base : ~0ull;  // first job of batch trace `lane`
        // the sample-generator key of every batch trace (tracegen.h tg_trace_key), one per lane, in shared memory
        s_tkey[threadIdx.x >> 5][lane] = tg_trace_key(P.seed, P.trace_id0 + t0 + lane);
        __syncwarp();
        const uint64_t gend = P.off[t0 + nb] - j_base;
        const uint64_t gbeg = __shfl_sync(FULL, my_off, 0);
        for (uint64_t c = gbeg; c < gend; c += 32) {
            if (P.dyn_only && c + 128 <= gend) {
                // mig_simulate's estimate: only DYNAMIC jobs need work; look 4 chunks ahead (4 loads in flight per
                // lane) and skip them when none is DYNAMIC, checking the records on the way
                uint4 r4[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) r4[u] = __ldg(P.jobs + c + 32 * u + lane);
                bool dyn = false, bad = false;
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const uint32_t cl = (r4[u].z >> 16) & 0xFFu;
                    dyn |= cl == kClassDynamic;
                    bad |= cl > 2 || (r4[u].z & 0xFFFFu) > 4096;
                }
                if (__any_sync(FULL, bad) && lane == 0) atomicOr(P.err, (unsigned long long)MIG_ERR_BAD_RECORD);
                if (!__any_sync(FULL, dyn)) {
                    c += 96;
                    continue;
                }
            }
            const uint64_t g = c + lane;
            const bool valid = g < gend;
            uint4 r = make_uint4(0, 0, 0, 0), e = make_uint4(0, 0, 0, 0);
            if (valid) {
                r = __ldg(P.jobs + g);
                if (P.ext) e = __ldg(P.ext + g);
            }
            const uint32_t cls = (r.z >> 16) & 0xFFu, T = r.z & 0xFFFFu;
            if (__any_sync(FULL, valid && (cls > 2 || T > 4096)) && lane == 0)
                atomicOr(P.err, (unsigned long long)MIG_ERR_BAD_RECORD);
            if (valid && cls != kClassDynamic && !P.dyn_only) {
                const uint64_t phys = (uint64_t)r.y + e.x + P.ctx;
                uint32_t fe[5], mfe[5];
#pragma unroll
                for (int l = 0; l < kMaxLevels; ++l) {
                    fe[l] = (l < (int)G.n_levels && T >= 1 && phys > G.level_mem[l]) ? 1u : kNever;
                    mfe[l] = fe[l] == 1u ? (uint32_t)phys : 0u;
                }
                store_estimate(P.out + g, r.x + e.x + P.ctx, 0, 0, G.n_levels, fe, 0.0, 0.0, 0.0, mfe, 0u,
                               (uint32_t)phys * T);
            }
            uint32_t dm = __ballot_sync(FULL, valid && cls == kClassDynamic);
            if (dm) {  // the generator keys of the chunk's 32 jobs at once (one lane each)
                // the batch trace holding record g: the last trace whose first job is <= g (offsets non-decreasing)
                uint32_t tb = 0;
#pragma unroll
                for (uint32_t step = 16; step; step >>= 1)
                    if (__shfl_sync(FULL, my_off, tb + step) <= g) tb += step;
                const uint32_t jt = (uint32_t)(g - __shfl_sync(FULL, my_off, tb));
                const uint64_t key = tg_job_key(s_tkey[threadIdx.x >> 5][tb], jt);  // = tg_key(seed, trace, jt)
                s_jkey[threadIdx.x >> 5][lane] = key;
                __syncwarp();
            }
            while (dm) {
                const uint32_t L = (uint32_t)__ffs(dm) - 1;
                dm &= dm - 1;
                const uint64_t gL = c + L;
                // the job's records again, one broadcast load each (L1 hits: the chunk just read them), so the chunk's
                // records are not kept live across the job loop
                const uint4 rr = __ldg(P.jobs + gL);
                const uint4 ee = P.ext ? __ldg(P.ext + gL) : make_uint4(0, 0, 0, 0);
                const uint2* rs = nullptr;
                uint32_t rcount = 0;
                if (P.samples) {
                    rs = P.samples + (P.sample_off[gL] - P.sample_off[0]);
                    const uint64_t cnt = P.sample_off[gL + 1] - P.sample_off[gL];
                    rcount = cnt > 0xFFFFu ? 0xFFFFu : (uint32_t)cnt;
                    if (rcount < (rr.z & 0xFFFFu)) {
                        if (lane == 0) atomicOr(P.err, (unsigned long long)MIG_ERR_BAD_RECORD);
                        if (rcount == 0) rs = nullptr;  // nothing recorded: fall back to the declared generator
                    }
                }
                estimate_dynamic<PLAIN>(G, P, s_jkey[threadIdx.x >> 5][L], rr, ee, lane, P.out + gL, rs, rcount);
            }
        }
    }
}

cudaError_t launch_estimate(const DevGeom& G, const mig_traces& tr, const mig_policy& pol, mig_job_estimate* out,
                            unsigned long long* scratch /* [counter, err] zeroed */, int sm_count,
                            bool dyn_only, cudaStream_t stream) {
    EstParams P;
    P.jobs = (const uint4*)tr.jobs;
    P.ext = (const uint4*)tr.jobs_ext;
    P.off = tr.trace_off;
    P.n_traces = tr.n_traces;
    P.trace_id0 = tr.trace_id0;
    P.seed = tr.seed;
    P.out = out;
    P.samples = (const uint2*)tr.samples;
    P.sample_off = tr.sample_off;
    P.counter = scratch;
    P.err = scratch + 1;
    P.ctx = pol.ctx_mib;
    P.eps_num = pol.eps_num;
    P.eps_den = pol.eps_den;
    P.conv_k = pol.conv_k;
    P.min_n = pol.min_n;
    P.z = pol.z;
    P.dyn_only = dyn_only ? 1u : 0u;
    P.ewma = (pol.flags & MIG_EWMA_REUSE) ? 1u : 0u;
    const int threads = 256;
    int per_sm = 0;
    const bool plain = !P.samples && !P.ewma;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, plain ? k_estimate<true> : k_estimate<false>, threads, 0);
    if (per_sm < 1) per_sm = 1;
    uint64_t want = (tr.n_traces + 8 * kEstBatch - 1) / (8 * kEstBatch);
    uint64_t blocks = (uint64_t)per_sm * sm_count;
    if (want < blocks) blocks = want;
    if (blocks < 1) blocks = 1;
    if (plain) k_estimate<true><<<(unsigned)blocks, threads, 0, stream>>>(G, P);
    else k_estimate<false><<<(unsigned)blocks, threads, 0, stream>>>(G, P);
    return cudaGetLastError();
}

}  // namespace mig
