"""Pins for the oracle's time-series predictor (Alg. 3 PeakMemoryPrediction).

Independent references: closed forms (constant / exactly linear series), numpy's least-squares (textbook two-pass
float OLS, np.polyfit), SPEC.md's worked values, a Monte-Carlo coverage property of the z bound, and the
early-restart analogue of PAPER.md:269/:763 (predict at iteration 6, OOM much later).
"""
import numpy as np
import pytest

from oracle import oracle as orc

Q1 = 65536  # inverse reuse ratio 1.0 in Q16


def test_constant_series():
    # [(1,100),(2,100),(3,100)] -> a=0, b=100, sigma=0
    P, phi, a, s = orc.fit_once([100, 100, 100], [Q1] * 3, T=3)
    assert (P, phi, a, s) == (100, 100.0, 0.0, 0.0)


def test_exact_linear_series():
    # (1,100)..(4,130) -> a=10, b=90, sigma=0; forecast at T: 10T+90 (exact)
    for T in [4, 20, 1000]:
        P, phi, a, s = orc.fit_once([100, 110, 120, 130], [Q1] * 4, T=T)
        assert a == 10.0 and s == 0.0 and phi == 10.0 * T + 90 and P == 10 * T + 90


def test_upper_bound_and_clamp():
    # sigma = 0 -> a*t+b; the bound is floored at 0 for a falling trend.
    P, phi, _, _ = orc.fit_once([100, 110, 120], [Q1] * 3, T=20)
    assert phi == 290.0
    P, phi, a, _ = orc.fit_once([60, 10, 2], [Q1] * 3, T=50)  # steeply falling -> negative forecast -> 0
    assert a < 0 and phi == 0.0 and P == 0


def test_reuse_ratio_division_spec_217():
    # mem (a=10,b=90), inverse reuse 1 + 0.05 t, T=20 -> (10*20+90)/(1+0.05*20) = 145 (rounded up).
    # Q16 slope 0.05*65536 = 3276.8 -> 3277.
    y = [10 * t + 90 for t in range(1, 6)]
    q = [Q1 + 3277 * t for t in range(1, 6)]
    P, phi, _, _ = orc.fit_once(y, q, T=20)
    want = 290.0 / ((Q1 + 3277 * 20) / Q1)
    assert abs(phi - want) < 1e-9 * want and P == 145


def test_matches_textbook_ols():
    # Exact-integer-moment OLS (R18) = numpy two-pass float OLS to <= 1e-9 relative.
    rng = np.random.default_rng(1234)
    for trial in range(200):
        n = int(rng.integers(3, 400))
        T = n + int(rng.integers(0, 600))
        t = np.arange(1, n + 1, dtype=np.float64)
        y = np.maximum(2, np.round(rng.uniform(500, 9000) + rng.uniform(-20, 80) * t +
                                   rng.normal(0, rng.uniform(1, 300), n))).astype(np.int64)
        qs = rng.integers(0, 200)
        q = (Q1 + qs * np.arange(1, n + 1)).astype(np.int64)
        z = 2.326
        P, phi, a, sig = orc.fit_once(y, q, T=T, pol=orc.policy(ctx_mib=0, z=z))
        A, B = np.polyfit(t, y.astype(np.float64), 1)
        resid = y - (A * t + B)
        sd = np.sqrt(np.sum(resid ** 2) / (n - 2))
        qa, qb = np.polyfit(t, q.astype(np.float64), 1)
        V = max((qa * T + qb) / Q1, 1.0)
        ref = max(A * T + B + z * sd, 0.0) / V
        assert a == pytest.approx(A, rel=1e-9, abs=1e-9)
        assert sig == pytest.approx(sd, rel=1e-7, abs=1e-6)  # sqrt of a cancellation-prone textbook SSR
        assert phi == pytest.approx(ref, rel=1e-9, abs=1e-6)
        if abs(ref - np.round(ref)) > 1e-6:
            assert P == int(np.ceil(ref))


def test_coverage_z_2326():
    # over 1000 seeded Gaussian-residual series the z=2.326 one-sided bound at the final
    # iteration covers the realised value in >= 97% of runs (99% nominal).
    rng = np.random.default_rng(7)
    hits = 0
    for _ in range(1000):
        n, T = 50, 60
        a, b, sd = rng.uniform(0, 50), rng.uniform(1000, 5000), rng.uniform(5, 200)
        t = np.arange(1, n + 1)
        y = np.round(b + a * t + rng.normal(0, sd, n)).astype(np.int64)
        _, phi, _, _ = orc.fit_once(y, [Q1] * n, T=T, pol=orc.policy(ctx_mib=0))
        realised = b + a * T + rng.normal(0, sd)
        hits += realised <= phi
    assert hits >= 970


def test_convergence_earliest_at_6_and_example_E():
    # Example E: req_i = 1000 + 100 i, invq = 1, T = 50: P_3..P_6 = 6000, converged at n = 6,
    # matching "predict ... at the 6th iteration" (R24).
    y = [1000 + 100 * i for i in range(1, 51)]
    e = orc.predict_series(y, [Q1] * 50, orc.policy(ctx_mib=0))
    assert e["conv_iter"] == 6 and e["pred_mib"] == 6000 and e["a"] == 100.0 and e["sigma"] == 0.0
    # + workspace + context
    e = orc.predict_series(y, [Q1] * 50, orc.policy(ctx_mib=512), ws=32)
    assert e["conv_iter"] == 6 and e["pred_mib"] == 6000 + 512 + 32


def test_convergence_rule_details():
    pol = orc.policy(ctx_mib=0)
    # short series: predictions need n >= 3, convergence needs 3 consecutive changes -> never before n = 6
    e = orc.predict_series([500] * 5, [Q1] * 5, pol)
    assert e["conv_iter"] == 0
    e = orc.predict_series([500] * 6, [Q1] * 6, pol)
    assert e["conv_iter"] == 6 and e["pred_mib"] == 500
    # a jump resets convergence: P changes by >= 1% at n = 7
    y = [500] * 6 + [900] + [900] * 20
    e = orc.predict_series(y, [Q1] * len(y), orc.policy(ctx_mib=0))
    assert e["conv_iter"] == 6  # already converged at 6; the predictor stops
    y = [500, 500, 500, 500, 900, 900, 900, 900, 900, 900, 900, 900]
    e = orc.predict_series(y, [Q1] * len(y), pol)
    assert e["conv_iter"] == 0 or e["conv_iter"] > 6


def test_reuse_lowers_physical_forecast():
    # a larger inverse reuse ratio (more reuse) means less physical memory.
    y = [1000 + 10 * i for i in range(1, 41)]
    e1 = orc.predict_series(y, [Q1] * 40, orc.policy(ctx_mib=0))
    e2 = orc.predict_series(y, [Q1 + 500 * i for i in range(1, 41)], orc.policy(ctx_mib=0))
    assert e2["pred_mib"] < e1["pred_mib"]


def test_prediction_error_at_ten_percent():
    # SPEC.md:480 / PAPER.md:765 analogue: the forecast made after 10% of the iterations is within 15% (mean
    # relative error) of the realised peak physical memory on the synthetic dynamic workloads (configs 3 and 4).
    from tracegen import tracegen as tg

    for cfg, n in [(3, 80), (4, 120)]:
        jobs, ext, off = tg.generate_host(cfg, n)
        seed = tg.seed_of(cfg)
        pol = orc.policy(ctx_mib=512)
        errs = []
        for t in range(n):
            for j in range(int(off[t]), int(off[t + 1])):
                if ((int(jobs[j, 2]) >> 16) & 0xFF) != 2:
                    continue
                T = int(jobs[j, 2]) & 0xFFFF
                y, q = tg.dyn_samples(seed, t, j - int(off[t]), jobs[j], ext[j], T)
                ws = int(ext[j, 0])
                peak = int((y.astype(np.int64) * 65536 // q).max()) + ws + 512
                P, _, _, _ = orc.fit_once(y[: max(3, T // 10)], q[: max(3, T // 10)], T, pol, ws)
                errs.append(abs(P - peak) / peak)
        assert len(errs) > 20 and np.mean(errs) <= 0.15, (cfg, np.mean(errs))


def test_recorded_series_equals_generated():
    # Recorded per-iteration samples fed explicitly give the same estimates as the generator.
    from tracegen import tracegen as tg

    jobs, ext, off = tg.generate_host(3, 60)
    seed = tg.seed_of(3)
    g = orc.Geometry(__import__("conftest").geom_path("a100-80gb"))
    smp, soff = tg.explicit_samples(jobs, ext, off, seed)
    a = orc.estimate(g, jobs, ext, off, orc.policy(), seed=seed)
    b = orc.estimate(g, jobs, ext, off, orc.policy(), seed=12345, samples=smp, sample_off=soff)
    dyn = ((jobs[:, 2] >> 16) & 0xFF) == 2
    assert dyn.sum() > 10
    assert np.array_equal(a[dyn], b[dyn])


def test_ewma_reuse_hand_derived():
    # MIG_EWMA_REUSE (reading R36; BASELINE.json north_star "least-squares and EWMA memory-forecast fit"): the inverse
    # reuse trend is replaced by L_1 = q_1, L_i = L_{i-1} + ((q_i - L_{i-1}) >> 3) (int64, arithmetic shift = floor),
    # V = max(L_n / 65536, 1). The L values below are worked by hand, not by the recurrence. y is constant 1000
    # (a = 0, sigma = 0), so phi = 1000 / V exactly as written and P = ceil(phi) (ctx = ws = 0).
    pol = orc.policy(ctx_mib=0, flags=orc.EWMA_REUSE)
    y = [1000, 1000, 1000]
    # rising: L1 = 65536; L2 = 65536 + 65536/8 = 73728; L3 = 73728 + (131072 - 73728)/8 = 73728 + 7168 = 80896
    P, phi, a, s = orc.fit_once(y, [65536, 131072, 131072], T=50, pol=pol)
    assert (a, s) == (0.0, 0.0)
    assert phi == pytest.approx(1000 * 65536 / 80896, rel=1e-12) and P == 811  # 810.1266 -> 811
    # falling, with floor (not truncation) of the negative differences:
    # L2 = 131072 + floor(-65535/8) = 131072 - 8192 = 122880; L3 = 122880 + floor(-57343/8) = 122880 - 7168 = 115712
    # (truncation would give 122881 and 115713)
    P, phi, _, _ = orc.fit_once(y, [131072, 65537, 65537], T=50, pol=pol)
    assert phi == pytest.approx(1000 * 65536 / 115712, rel=1e-12) and P == 567  # 566.3717 -> 567
    assert phi != pytest.approx(1000 * 65536 / 115713, rel=1e-9)
    # n = 4 extends the same hand sequence: L4 = 115712 + floor((65537 - 115712)/8) = 115712 + floor(-6271.875)
    # = 115712 - 6272 = 109440
    P, phi, _, _ = orc.fit_once(y + [1000], [131072, 65537, 65537, 65537], T=50, pol=pol)
    assert phi == pytest.approx(1000 * 65536 / 109440, rel=1e-12) and P == 599  # 598.83 -> 599
    # below 1.0 the ratio is clamped (V >= 1): phi = u
    P, phi, _, _ = orc.fit_once(y, [32768, 32768, 32768], T=50, pol=pol)
    assert phi == 1000.0 and P == 1000
    # the EWMA is a level, not a trend: the OLS line through [65536, 66536, 67536] is 64536 + 1000 t, which at
    # T = 50 divides by 114536 / 65536 = 1.7477; the EWMA is L = 65536, 65661, 65895 -> 1.00548
    P, phi, _, _ = orc.fit_once(y, [65536, 66536, 67536], T=50, pol=pol)
    assert phi == pytest.approx(1000 * 65536 / 65895, rel=1e-12) and P == 995  # 994.55 -> 995
    P_ols, _, _, _ = orc.fit_once(y, [65536, 66536, 67536], T=50, pol=orc.policy(ctx_mib=0))
    assert P_ols == 573  # 1000 * 65536 / 114536 = 572.18 -> 573
