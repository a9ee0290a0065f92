/* tracegen.h — seeded synthetic job-queue ("trace") generator.
 *
 * INPUT GENERATION ONLY. This module is the one piece of code that both the CPU oracle (oracle/) and the CUDA path
 * (paper_2508_18556_b200/csrc) may use: it draws the synthetic workloads and the per-iteration memory samples a
 * dynamic job would report ("collect requested memory req_mem and reuse_ratio through instrumented
 * PyTorch"). It holds NONE of the method's arithmetic: no tight-fit, no placement, no reachability, no regression,
 * no OOM test, no scheduling. Everything here is integer-only (splitmix64 counters, mulhi range reduction,
 * Irwin-Hall noise) so host and device produce bit-identical traces.
 *
 * Trace format:
 *   jobs[j] (4 x u32):
 *     x = est_mib   (STATIC/MODEL: compile-time or model-size estimate)   | b_mib  (DYNAMIC: intercept)
 *     y = true_mib  (STATIC/MODEL: true footprint excl. ws/ctx)                                | q0_q16 (DYNAMIC: inverse reuse at t=0, Q16)
 *     z = iters (bits 0..15) | class (bits 16..23) | flags (bits 24..31, reserved = 0)
 *     w = iter_ticks (1 tick = 1 ms)
 *   ext[j] (4 x u32, optional; all-zero when absent):
 *     x = ws_mib (third-party workspace)
 *     y = warps  (compile-time warp count)
 *     z = slope_q8 (MiB/iter in Q8)                                                        (DYNAMIC only)
 *     w = sigma_mib (bits 0..15) | qslope_q16 (bits 16..31, inverse-reuse slope, Q16)      (DYNAMIC only)
 *   trace_off[t] (u64): CSR offsets, n_traces + 1 entries.
 */
#ifndef TRACEGEN_H
#define TRACEGEN_H

#include <stdint.h>

#ifdef __CUDACC__
#define TG_HD __host__ __device__ __forceinline__
#else
#define TG_HD static inline
#endif

#define TG_CLASS_STATIC 0u
#define TG_CLASS_MODEL 1u
#define TG_CLASS_DYNAMIC 2u

#define TG_SEED(c) (0x4D49474D00000000ull + (uint64_t)(c))
#define TG_GOLDEN 0x9E3779B97F4A7C15ull
#define TG_MAX_JOBS_PER_TRACE 128u

/* splitmix64 finaliser (Steele, Lea, Flood 2014). */
TG_HD uint64_t tg_mix64(uint64_t x) {
    x += TG_GOLDEN;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

/* Counter-based stream key for (seed, trace, job). job = 0xFFFFFFFF names the trace-level stream. */
TG_HD uint64_t tg_trace_key(uint64_t seed, uint64_t trace) { return tg_mix64(seed ^ tg_mix64(trace)); }
TG_HD uint64_t tg_job_key(uint64_t trace_key, uint32_t job) { return tg_mix64(trace_key + (uint64_t)job * TG_GOLDEN); }
TG_HD uint64_t tg_key(uint64_t seed, uint64_t trace, uint32_t job) {
    return tg_job_key(tg_trace_key(seed, trace), job);
}

/* Draw number ctr of a stream. */
TG_HD uint64_t tg_draw(uint64_t key, uint64_t ctr) { return tg_mix64(key + ctr * TG_GOLDEN); }

/* Uniform integer in [0, n) from the high 32 bits (mulhi range reduction). n >= 1. */
TG_HD uint32_t tg_uni(uint64_t r, uint32_t n) { return (uint32_t)(((r >> 32) * (uint64_t)n) >> 32); }

/* Uniform integer in [lo, hi] inclusive. */
TG_HD uint32_t tg_range(uint64_t r, uint32_t lo, uint32_t hi) { return lo + tg_uni(r, hi - lo + 1u); }

/* "Octave-uniform" integer in [2^a, 2^b): exponent uniform in [a, b), then uniform inside the octave. */
TG_HD uint32_t tg_octave(uint64_t r, uint32_t a, uint32_t b) {
    uint32_t e = a + tg_uni(r, b - a);
    return (1u << e) + (uint32_t)(((r & 0xFFFFFFFFull) * (uint64_t)(1u << e)) >> 32);
}

/* 32-bit integer hash ("lowbias32", C. Wellons 2018: two multiplies, three xorshifts). */
TG_HD uint32_t tg_hash32(uint32_t x) {
    x ^= x >> 16;
    x *= 0x7feb352du;
    x ^= x >> 15;
    x *= 0x846ca68bu;
    x ^= x >> 16;
    return x;
}

/* The 32 random bits of iteration i of a DYNAMIC job's sample stream: one counter hash keyed by both halves of the
 * job's splitmix64 key. The per-iteration draw is the hot part of generating a series in-kernel (SURVEY.md §8(d)
 * budgets ~15 ops for RNG + Irwin-Hall per iteration): one hash, ~10 32-bit instructions. */
TG_HD uint32_t tg_iter_bits(uint64_t job_key, uint32_t i) {
    return tg_hash32(((uint32_t)job_key ^ (i * 0x9E3779B9u)) + (uint32_t)(job_key >> 32));
}

/* Irwin-Hall(4) noise with standard deviation ~sigma from the four bytes of r: (sum of four 8-bit uniforms - 510)
 * * 256 has standard deviation 37837.6 = 2^28 / 7094.3, so noise = floor((sum - 510) * 256 * (sigma * 7094) / 2^28),
 * written as the high word of 4096 (sum - 510) * (sigma * 7094) (|4096 (sum - 510)| < 2^21; sigma < 2^16): one
 * 32x32->64 multiply. |noise| <= 510 * 65535 * 7094 / 2^20 < 2^18. The byte sum is one dp4a on the device. No
 * log/cos/division, so host and device are bit-identical. */
TG_HD int32_t tg_irwin_hall(uint32_t r, uint32_t sigma) {
#ifdef __CUDA_ARCH__
    const int32_t s = (int32_t)__dp4a(r, 0x01010101u, 0u);
    /* the high word of the signed 64-bit product: one IMAD.HI */
    return __mulhi((s - 510) * 4096, (int32_t)((sigma & 0xFFFFu) * 7094u));
#else
    const int32_t s = (int32_t)((r & 0xFFu) + ((r >> 8) & 0xFFu) + ((r >> 16) & 0xFFu) + (r >> 24));
    return (int32_t)(((int64_t)((s - 510) * 4096) * (int64_t)(int32_t)((sigma & 0xFFFFu) * 7094u)) >> 32);
#endif
}

/* Per-iteration sample i (1-based) of a DYNAMIC job: requested MiB y_i (allocator-rounded up to 2 MiB, >= 2) and
 * inverse reuse ratio q_i in Q16 (inv_reuse = 1/reuse_ratio >= 1). */
TG_HD void tg_dyn_sample(uint64_t job_key, uint32_t i, uint32_t b_mib, uint32_t slope_q8, uint32_t sigma_mib,
                         uint32_t q0_q16, uint32_t qslope_q16, uint32_t* y, uint32_t* q) {
    int64_t v = (int64_t)b_mib + (int64_t)(((uint64_t)slope_q8 * i) >> 8) +
                (int64_t)tg_irwin_hall(tg_iter_bits(job_key, i), sigma_mib);
    if (v < 2) v = 2;
    v = (v + 1) & ~(int64_t)1;
    *y = (uint32_t)v;
    *q = q0_q16 + qslope_q16 * i;
}

/* tg_dyn_sample in 32-bit arithmetic, for series whose bounds keep every intermediate in range: b + (slope_q8 * T
 * >> 8) + 2^19 < 2^31 and slope_q8 * T < 2^32 (the Irwin-Hall noise is below 2^18 in magnitude). Equal to
 * tg_dyn_sample for every i <= T under those bounds (tests/test_tracegen.py). */
TG_HD void tg_dyn_sample_fast(uint64_t job_key, uint32_t i, uint32_t b_mib, uint32_t slope_q8, uint32_t sigma_mib,
                              uint32_t q0_q16, uint32_t qslope_q16, uint32_t* y, uint32_t* q) {
    int32_t v = (int32_t)(b_mib + ((slope_q8 * i) >> 8)) + tg_irwin_hall(tg_iter_bits(job_key, i), sigma_mib);
    v = v < 2 ? 2 : v;
    v = (v + 1) & ~1;
    *y = (uint32_t)v;
    *q = q0_q16 + qslope_q16 * i;
}

/* ---------------------------------------------------------------------------------------------------------------
 * Config generators. cfg 2..5; cfg 1 is the fixed hand-worked trace (tests/golden).
 * ------------------------------------------------------------------------------------------------------------- */

TG_HD uint32_t tg_jobs_per_trace(uint32_t cfg) {
    return cfg == 2 ? 100u : cfg == 3 ? 20u : cfg == 4 ? 4u : cfg == 5 ? 50u : 0u;
}
TG_HD uint32_t tg_has_ext(uint32_t cfg) { return cfg == 3 || cfg == 4 || cfg == 5; }

/* Exact bucket counts for ratio r[4] scaled to J jobs (largest remainder, ties to the lower bucket), then a
 * Fisher-Yates shuffle driven by the trace stream. out[j] = bucket of job j. */
TG_HD void tg_mix_buckets(uint64_t tkey, const uint32_t r[4], uint32_t J, uint8_t* out) {
    uint32_t tot = r[0] + r[1] + r[2] + r[3];
    uint32_t cnt[4], rem[4], used = 0;
    for (int k = 0; k < 4; ++k) {
        cnt[k] = r[k] * J / tot;
        rem[k] = r[k] * J % tot;
        used += cnt[k];
    }
    while (used < J) {
        int best = -1;
        for (int k = 0; k < 4; ++k)
            if (r[k] && (best < 0 || rem[k] > rem[best])) best = k;
        cnt[best] += 1;
        rem[best] = 0;
        used += 1;
    }
    uint32_t j = 0;
    for (int k = 0; k < 4; ++k)
        for (uint32_t c = 0; c < cnt[k]; ++c) out[j++] = (uint8_t)k;
    for (uint32_t i = J - 1; i >= 1; --i) {
        uint32_t k = tg_uni(tg_draw(tkey, 100u + i), i + 1u);
        uint8_t t = out[i];
        out[i] = out[k];
        out[k] = t;
    }
}

/* Rodinia-style bucket true footprint (MiB, excl. the 512 MiB context): small (256,4608], medium (4608,9728],
 * large (9728,19968], full (19968,40448] — the 5/10/20/40 GB buckets of PAPER.md:641-646. */
TG_HD uint32_t tg_rodinia_true(uint64_t r, uint32_t bucket) {
    const uint32_t lo[4] = {256u, 4608u, 9728u, 19968u};
    const uint32_t hi[4] = {4608u, 9728u, 19968u, 40448u};
    return lo[bucket] + 1u + tg_uni(r, hi[bucket] - lo[bucket]);
}

TG_HD void tg_put(uint32_t* jobs, uint32_t* ext, uint32_t j, uint32_t x, uint32_t y, uint32_t iters, uint32_t cls,
                  uint32_t ticks, uint32_t ws, uint32_t warps, uint32_t slope_q8, uint32_t sigma, uint32_t qslope) {
    jobs[4 * j + 0] = x;
    jobs[4 * j + 1] = y;
    jobs[4 * j + 2] = (iters & 0xFFFFu) | (cls << 16);
    jobs[4 * j + 3] = ticks;
    if (ext) {
        ext[4 * j + 0] = ws;
        ext[4 * j + 1] = warps;
        ext[4 * j + 2] = slope_q8;
        ext[4 * j + 3] = (sigma & 0xFFFFu) | (qslope << 16);
    }
}

/* LLM KV-growth dynamic job whose requested + ctx memory crosses `cap_mib` at about iteration i_x
 * (OOM at batch 94 / 72 on a 10 GB slice). */
TG_HD void tg_llm_job(uint64_t jkey, uint32_t* jobs, uint32_t* ext, uint32_t j, uint32_t cap_mib, uint32_t ctx,
                      uint32_t b_lo, uint32_t b_hi, uint32_t ix_lo, uint32_t ix_hi, uint32_t t_hi, uint32_t qslope_hi,
                      uint32_t ws) {
    uint32_t b = tg_range(tg_draw(jkey, 0x10001u), b_lo, b_hi);
    uint32_t ix = tg_range(tg_draw(jkey, 0x10002u), ix_lo, ix_hi);
    uint32_t T = tg_range(tg_draw(jkey, 0x10003u), ix + 20u, t_hi);
    uint32_t gap = cap_mib - ctx - ws - b;
    uint32_t slope_q8 = (uint32_t)((((uint64_t)gap << 8) + ix - 1u) / ix);
    uint32_t sigma = b / 200u;
    uint32_t qs = qslope_hi ? tg_uni(tg_draw(jkey, 0x10004u), qslope_hi + 1u) : 0u;
    uint32_t ticks = tg_octave(tg_draw(jkey, 0x10005u), 5u, 8u);
    tg_put(jobs, ext, j, b, 65536u, T, TG_CLASS_DYNAMIC, ticks, ws, 0u, slope_q8, sigma, qs);
}

/* ML training job (DNNMem-estimated MODEL class): est = true*(100+e)/100, e in [-15, +10]. */
TG_HD void tg_model_job(uint64_t jkey, uint32_t* jobs, uint32_t* ext, uint32_t j, uint32_t lo, uint32_t hi,
                        uint32_t ws) {
    uint32_t tru = lo + 1u + tg_uni(tg_draw(jkey, 0x10001u), hi - lo);
    uint32_t e = tg_uni(tg_draw(jkey, 0x10002u), 26u);
    uint32_t est = (uint32_t)(((uint64_t)tru * (85u + e)) / 100u);
    uint32_t iters = tg_range(tg_draw(jkey, 0x10003u), 50u, 400u);
    uint32_t ticks = tg_octave(tg_draw(jkey, 0x10004u), 7u, 10u);
    tg_put(jobs, ext, j, est, tru, iters, TG_CLASS_MODEL, ticks, ws, 0u, 0u, 0u, 0u);
}

/* ML dynamic-memory training job (FLAN-T5-train-like): linear growth, noisy, reuse improving. */
TG_HD void tg_mldyn_job(uint64_t jkey, uint32_t* jobs, uint32_t* ext, uint32_t j, uint32_t ws) {
    uint32_t b = tg_range(tg_draw(jkey, 0x10001u), 2048u, 6144u);
    uint32_t slope_q8 = tg_range(tg_draw(jkey, 0x10002u), 8u * 256u, 64u * 256u);
    uint32_t T = tg_range(tg_draw(jkey, 0x10003u), 60u, 400u);
    uint32_t sigma = tg_range(tg_draw(jkey, 0x10004u), 16u, 128u);
    uint32_t qs = tg_uni(tg_draw(jkey, 0x10005u), 65u);
    uint32_t ticks = tg_octave(tg_draw(jkey, 0x10006u), 7u, 10u);
    tg_put(jobs, ext, j, b, 65536u, T, TG_CLASS_DYNAMIC, ticks, ws, 0u, slope_q8, sigma, qs);
}

/* Rodinia STATIC job: est = true except 1/64 of jobs get est = 3/4 true (seeds OOM restarts). */
TG_HD void tg_rodinia_job(uint64_t jkey, uint32_t* jobs, uint32_t* ext, uint32_t j, uint32_t tru, uint32_t ticks) {
    uint64_t r = tg_draw(jkey, 0x10001u);
    uint32_t est = ((r & 63u) == 0u) ? (uint32_t)(((uint64_t)tru * 3u) / 4u) : tru;
    tg_put(jobs, ext, j, est, tru, 8u, TG_CLASS_STATIC, ticks, 0u, 0u, 0u, 0u, 0u);
}

/* Generate trace `trace` of config cfg into jobs/ext (tg_jobs_per_trace(cfg) records). Returns the job count. */
TG_HD uint32_t tg_gen_trace(uint32_t cfg, uint64_t seed, uint64_t trace, uint32_t* jobs, uint32_t* ext) {
    const uint32_t J = tg_jobs_per_trace(cfg);
    const uint64_t tkey = tg_key(seed, trace, 0xFFFFFFFFu);
    uint8_t bucket[TG_MAX_JOBS_PER_TRACE];
    if (cfg == 2) {
        /* 7 Rodinia mixes: Hm1-3 small, Hm4 large, Ht1 11:2:2:0, Ht2 1:0:1:1, Ht3 4:0:1:1. */
        const uint32_t R[7][4] = {{1, 0, 0, 0}, {1, 0, 0, 0}, {1, 0, 0, 0}, {0, 0, 1, 0},
                                  {11, 2, 2, 0}, {1, 0, 1, 1}, {4, 0, 1, 1}};
        uint32_t mix = tg_uni(tg_draw(tkey, 1u), 7u);
        tg_mix_buckets(tkey, R[mix], J, bucket);
        /* Homogeneous mixes run one benchmark: one archetype (footprint, iteration time) per trace. */
        uint32_t arch_true = tg_rodinia_true(tg_draw(tkey, 2u), bucket[0]);
        uint32_t arch_ticks = tg_octave(tg_draw(tkey, 3u), 6u, 11u);
        for (uint32_t j = 0; j < J; ++j) {
            uint64_t jkey = tg_key(seed, trace, j);
            uint32_t tru = mix < 4 ? arch_true : tg_rodinia_true(tg_draw(jkey, 0x10002u), bucket[j]);
            uint32_t ticks = mix < 4 ? arch_ticks : tg_octave(tg_draw(jkey, 0x10003u), 6u, 11u);
            tg_rodinia_job(jkey, jobs, ext, j, tru, ticks);
        }
    } else if (cfg == 3) {
        /* ML mixes Ml1 1:0:1:0, Ml2 1:0:0:0, Ml3 0:0:1:0 plus 25% dynamic-memory jobs. */
        const uint32_t R[3][4] = {{1, 0, 1, 0}, {1, 0, 0, 0}, {0, 0, 1, 0}};
        uint32_t mix = tg_uni(tg_draw(tkey, 1u), 3u);
        tg_mix_buckets(tkey, R[mix], J, bucket);
        for (uint32_t j = 0; j < J; ++j) {
            uint64_t jkey = tg_key(seed, trace, j);
            if ((tg_draw(jkey, 0x10000u) & 3u) == 0u)
                tg_mldyn_job(jkey, jobs, ext, j, 32u);
            else if (bucket[j] == 0)
                tg_model_job(jkey, jobs, ext, j, 3072u, 9216u, 32u);
            else
                tg_model_job(jkey, jobs, ext, j, 12288u, 19456u, 32u);
        }
    } else if (cfg == 4) {
        /* Homogeneous LLM inference mixes: FLAN-T5 / Qwen2 / Llama-3 KV growth, 10 GB slice
         * crossed near iteration 27 / 94 / 72. */
        uint32_t arch = tg_uni(tg_draw(tkey, 1u), 3u);
        for (uint32_t j = 0; j < J; ++j) {
            uint64_t jkey = tg_key(seed, trace, j);
            if (arch == 0)
                tg_llm_job(jkey, jobs, ext, j, 10240u, 512u, 3072u, 5120u, 24u, 48u, 300u, 0u, 0u);
            else if (arch == 1)
                tg_llm_job(jkey, jobs, ext, j, 10240u, 512u, 5120u, 8192u, 72u, 100u, 1000u, 0u, 0u);
            else
                tg_llm_job(jkey, jobs, ext, j, 10240u, 512u, 4096u, 7168u, 56u, 80u, 1000u, 0u, 0u);
        }
    } else if (cfg == 5) {
        /* Policy-sweep mix: 60% Rodinia STATIC (buckets 4:2:1:1), 25% MODEL scaled to 40 GB, 15% LLM DYNAMIC
         * crossing the 5 GB slice in [20, 100] iterations. */
        for (uint32_t j = 0; j < J; ++j) {
            uint64_t jkey = tg_key(seed, trace, j);
            uint32_t u = tg_uni(tg_draw(jkey, 0x10000u), 100u);
            if (u < 60u) {
                uint32_t w = tg_uni(tg_draw(jkey, 0x10007u), 8u);
                uint32_t bk = w < 4u ? 0u : w < 6u ? 1u : w < 7u ? 2u : 3u;
                uint32_t tru = tg_rodinia_true(tg_draw(jkey, 0x10002u), bk);
                uint32_t ticks = tg_octave(tg_draw(jkey, 0x10003u), 6u, 11u);
                tg_rodinia_job(jkey, jobs, ext, j, tru, ticks);
            } else if (u < 85u) {
                if (tg_draw(jkey, 0x10008u) & 1u)
                    tg_model_job(jkey, jobs, ext, j, 1536u, 4608u, 32u);
                else
                    tg_model_job(jkey, jobs, ext, j, 6144u, 9728u, 32u);
            } else {
                tg_llm_job(jkey, jobs, ext, j, 5120u, 512u, 1536u, 3072u, 20u, 100u, 200u, 16u, 0u);
            }
        }
    }
    return J;
}

#endif /* TRACEGEN_H */
