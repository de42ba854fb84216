"""Pins for the CPU oracle against what the paper and the mathematics fix.

Every test here runs on CPU (no GPU marker).  Each one is chosen so that a
plausible mistake in the oracle (a dropped term, a wrong sign or index, a
transposed operand, a shifted tap) fails at least one of them.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle
from oracle import bruteforce, mulaw, perfmodel
from paper_1702_07825_b200 import synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_numbers.json")))


def tiny(L, r, s, a=16, dil=None, seed=0, scale=1.0):
    cfg = synth.Config(L, r, s, a, tuple(dil) if dil else None)
    w = synth.make_weights(cfg, seed) * np.float32(scale)
    return cfg, w.astype(np.float32)


def run_tf(cfg, w, cond, hop, codes, **kw):
    return oracle.run(cfg.n_layers, cfg.residual, cfg.skip, w, cond, hop, len(codes),
                      forced=codes, levels=cfg.levels, dilations=cfg.dilation_list(), **kw)


# ---------------------------------------------------------------- mu-law (R14)
def test_mulaw_matches_torchaudio():
    torchaudio = pytest.importorskip("torchaudio")
    import torch
    x = np.linspace(-1.0, 1.0, 20001)
    ours = mulaw.encode(x)
    ref = torchaudio.functional.mu_law_encoding(torch.from_numpy(x), 256).numpy()
    assert np.array_equal(ours, ref)
    c = np.arange(256)
    ref_dec = torchaudio.functional.mu_law_decoding(torch.from_numpy(c), 256).numpy()
    np.testing.assert_allclose(mulaw.decode(c), ref_dec, rtol=0, atol=1e-6)


def test_mulaw_endpoints_idempotence_and_silence_code():
    assert mulaw.encode(-1.0) == 0 and mulaw.encode(1.0) == 255
    assert mulaw.encode(0.0) == 128  # the silence code used for negative times (R4)
    c = np.arange(256)
    assert np.array_equal(mulaw.encode(mulaw.decode(c)), c)
    x = np.linspace(-1, 1, 10001)
    assert np.all(np.diff(mulaw.encode(x)) >= 0)
    # quantisation bound: half a level is 1/mu in the companded domain, and the
    # inverse map's slope ln(1+mu)(1+mu|x|)/mu grows by at most (1+mu)^(1/mu) over it
    mu = 255
    err = np.abs(mulaw.decode(mulaw.encode(x)) - x)
    bound = (1 + mu * np.abs(x)) * np.log1p(mu) / mu**2 * (1 + mu) ** (1 / mu) + 1e-12
    assert np.all(err <= bound)


# ---------------------------------------------------- App. E / §5 printed numbers
def test_parameter_count_and_megabytes():
    n = perfmodel.n_params(40, 64, 256)
    assert n == 1_646_912
    assert abs(n - GOLD["params_l40_r64_s256"]["value"]) / 1.6e6 < 0.05
    assert abs(n * 4 / 1e6 - GOLD["megabytes_fp32_l40_r64_s256"]["value"]) / 6.4 < 0.05
    # three independent roster counts agree: App. E formula, synth roster, C oracle
    for L, r, s in [(40, 64, 256), (20, 64, 128), (20, 64, 256), (20, 128, 256), (3, 5, 7)]:
        n = perfmodel.n_params(L, r, s)
        assert synth.weights_numel(synth.Config(L, r, s)) == n
        assert oracle.weights_numel(L, r, s, 256) == n


def test_app_e_cost_model_matches_printed_values():
    per_layer = perfmodel.cost_layer(64)
    assert per_layer == 44_224
    assert abs(per_layer - GOLD["flops_per_layer_l40_r64"]["value"]) / 42e3 < 0.06  # R18
    per_second = perfmodel.cost_sample(40, 64, 256) * 16384
    assert perfmodel.cost_sample(40, 64, 256) == 3_348_992
    assert abs(per_second - GOLD["flops_per_audio_second_l40_r64_s256"]["value"]) / 55e9 < 0.01
    # weights re-read once per sample at 16,384 Hz (~100 GB/s)
    gbs = perfmodel.n_params(40, 64, 256) * 4 * 16384 / 1e9
    assert abs(gbs - GOLD["weight_reload_gb_per_s"]["value"]) / 100 < 0.1
    # real-time budget 60 us/sample at 16 kHz, 1.5 us/layer at l=40
    assert abs(1e6 / 16384 - GOLD["us_per_sample_16khz"]["value"]) / 60 < 0.05
    assert abs(1e6 / 16384 / 40 - GOLD["us_per_layer_l40"]["value"]) / 1.5 < 0.05


# ---------------------------------------------------- receptive field (R2)
def test_receptive_field_reading_reproduces_paper():
    R40 = perfmodel.receptive_field(oracle.default_dilations(40))
    R20 = perfmodel.receptive_field(oracle.default_dilations(20))
    assert R40 == 4094 and R20 == 2048
    ms = R40 / 48000 * 1e3
    assert abs(ms - GOLD["receptive_field_ms_l40_48khz"]["value"]) / 83 < 0.05
    assert abs(R20 / R40 - GOLD["receptive_field_ratio_l20_l40"]["value"]) < 0.01
    # only a cycle of 10 is consistent with 83 ms (cycles 9 and 11 are far off)
    for c in (9, 11):
        R = 2 + sum(1 << (j % c) for j in range(40))
        assert abs(R / 48 - 83) / 83 > 0.4
    assert perfmodel.receptive_field([1]) == 3
    assert perfmodel.receptive_field(oracle.default_dilations(10)) == 1025


def _subset_sums(d):
    sums = {0}
    for x in d:
        sums |= {v + x for v in sums}
    return sums


@pytest.mark.parametrize("dil", [[1], [3], [3, 1], [1, 2, 4], [5, 5]])
def test_exact_lag_set_by_perturbation(dil):
    """logits[n] depends on codes[m] iff n - m in {1, 2} + SubsetSums(d)."""
    cfg, w = tiny(len(dil), 4, 6, a=16, dil=dil, seed=3, scale=3.0)
    N, hop = 40, 4
    cond = synth.make_cond(cfg, synth.n_frames_for(N, hop), 1)
    codes = synth.make_codes(N, 5, cfg.levels)
    _, base, _ = run_tf(cfg, w, cond, hop, codes)
    lags = {1 + v for v in _subset_sums(dil)} | {2 + v for v in _subset_sums(dil)}
    m = 10
    pert = codes.copy()
    pert[m] = (pert[m] + 7) % cfg.levels
    _, lg, _ = run_tf(cfg, w, cond, hop, pert)
    for n in range(N):
        changed = not np.array_equal(lg[n], base[n])
        assert changed == ((n - m) in lags), (n, n - m, sorted(lags))


def test_default_schedule_lag_set_is_exactly_1_to_R():
    """l = 20, c = 10: the lag set is exactly {1..2048} = R (S:71 + PAPER.md:166)."""
    sums = _subset_sums(oracle.default_dilations(20))
    lags = {1 + v for v in sums} | {2 + v for v in sums}
    assert lags == set(range(1, 2049))


def test_causality_in_conditioning():
    cfg, w = tiny(3, 4, 6, a=16, dil=[1, 2, 4], seed=4)
    N, hop = 48, 4
    cond = synth.make_cond(cfg, synth.n_frames_for(N, hop), 2)
    codes = synth.make_codes(N, 6, cfg.levels)
    _, base, _ = run_tf(cfg, w, cond, hop, codes)
    for f in (0, 3, 7):
        c2 = cond.copy()
        c2[f] += 0.25
        _, lg, _ = run_tf(cfg, w, c2, hop, codes)
        assert np.array_equal(lg[: f * hop], base[: f * hop])
        assert not np.array_equal(lg[f * hop], base[f * hop])


# ---------------------------------------------------- two independent oracles
@pytest.mark.parametrize("seed", range(10))
def test_ring_oracle_equals_bruteforce_teacher_forced(seed):
    rng = np.random.default_rng(seed)
    dil = [[3], [5, 5], [3, 1], [1, 2, 4], [2, 1, 3, 7]][seed % 5]
    r = int(rng.choice([3, 4, 8]))
    cfg, w = tiny(len(dil), r, 5 + seed % 3, a=16, dil=dil, seed=seed)
    N, hop = 256, int(rng.choice([1, 3, 16]))
    cond = synth.make_cond(cfg, synth.n_frames_for(N, hop), seed)
    codes = synth.make_codes(N, seed, cfg.levels)
    _, lg, _ = run_tf(cfg, w, cond, hop, codes)
    bf = bruteforce.forward_logits(w, cfg.n_layers, r, cfg.skip, codes, cond, hop, cfg.levels, dil)
    assert np.max(np.abs(lg - bf)) <= 1e-12


@pytest.mark.parametrize("seed", range(3))
def test_ring_oracle_equals_bruteforce_free_running(seed):
    dil = [[1, 2, 4], [5, 5], [3, 1]][seed]
    cfg, w = tiny(len(dil), 4, 6, a=16, dil=dil, seed=seed, scale=4.0)
    N, hop = 64, 8
    cond = synth.make_cond(cfg, synth.n_frames_for(N, hop), seed)
    u = synth.make_uniforms(N, seed)
    codes, _, _ = oracle.run(cfg.n_layers, 4, 6, w, cond, hop, N, uniforms=u, levels=16,
                             dilations=dil)
    bf = bruteforce.generate(w, cfg.n_layers, 4, 6, cond, hop, u, N, 16, dil)
    assert np.array_equal(codes, bf)
    assert len(set(codes.tolist())) > 4  # not a degenerate trajectory


# ---------------------------------------------------- closed-form special cases
def test_zero_weights_give_floor_256u():
    """All-zero weights => logits = 0 => p uniform => y = floor(256 u) exactly."""
    cfg = synth.C1
    w = np.zeros(synth.weights_numel(cfg), np.float32)
    N, hop = 300, 64
    cond = synth.make_cond(cfg, synth.n_frames_for(N, hop), 0)
    u = synth.make_uniforms(N, 0)
    codes, lg, _ = oracle.run(20, 64, 128, w, cond, hop, N, uniforms=u)
    assert np.all(lg == 0.0)
    assert np.array_equal(codes, np.floor(256 * u.astype(np.float64)).astype(np.uint8))


def test_one_hot_logits_fix_the_code():
    cfg = synth.Config(2, 8, 16)
    w = synth.make_weights(cfg, 1)
    P = synth.split_weights(cfg, w)
    P["B_out"][:] = 0
    P["B_out"][42] = 1e4
    P["W_out"][:] = 0
    N = 50
    cond = synth.make_cond(cfg, N, 0)
    codes, _, _ = oracle.run(2, 8, 16, w, cond, 1, N, uniforms=synth.make_uniforms(N, 0),
                             dilations=cfg.dilation_list())
    assert np.all(codes == 42)


def test_bias_only_head_gives_closed_form_draws():
    """Only B_out nonzero => logits = B_out; codes are inverse-CDF draws from softmax(B_out)."""
    cfg = synth.Config(3, 8, 16)
    w = synth.make_weights(cfg, 2, "peaky")
    P = synth.split_weights(cfg, w)
    bout = P["B_out"].copy()
    w[:] = 0
    P["B_out"][:] = bout
    N = 400
    u = synth.make_uniforms(N, 9)
    codes, lg, _ = oracle.run(3, 8, 16, w, synth.make_cond(cfg, N, 0), 1, N, uniforms=u,
                              dilations=cfg.dilation_list())
    assert np.all(lg == bout.astype(np.float64)[None, :])
    p = np.exp(bout.astype(np.float64) - bout.max())
    cdf = np.cumsum(p) / p.sum()
    expect = np.array([int(np.argmax(cdf > float(x))) for x in u])
    assert np.array_equal(codes, expect)


@pytest.mark.parametrize("gain", [1.0, 50.0, 400.0])
def test_softmax_pinned_to_library_and_draw_frequencies(gain):
    """p = softmax(l) as the oracle's sampler forms it: equal to
    scipy.special.softmax (a library routine, not a retyped formula), summing to 1 in fp64,
    and the inverse-CDF draw (reading R11) realises exactly these
    probabilities: over the grid u_i = (i + 1/2) / G the count of draws of code k is
    within 1 of G p_k (the draws of k are the u in [P_{k-1}/S, P_k/S), an interval of
    length p_k).  A dropped max shift, a wrong comparison or an off-by-one in the scan
    fails one of these."""
    from scipy.special import softmax as sp_softmax
    lg = synth.make_weights(synth.Config(1, 2, 2), 3)[:256].astype(np.float64) * gain
    p = oracle.softmax(lg)
    assert abs(p.sum() - 1.0) < 1e-12
    np.testing.assert_allclose(p, sp_softmax(lg), rtol=1e-12, atol=1e-300)
    G = 20000
    grid = (np.arange(G) + 0.5) / G
    draws = np.array([oracle.sample(lg, np.float32(x)) for x in grid])
    counts = np.bincount(draws, minlength=256)
    assert np.all(np.abs(counts - G * p) <= 1.0 + 1e-6 * G), np.max(np.abs(counts - G * p))
    assert np.all(draws[1:] >= draws[:-1])  # monotone in u


def test_sampler_edges():
    lg = synth.make_weights(synth.Config(1, 2, 2), 0)[:256].astype(np.float64) * 50
    # u = 0 picks the first code with nonzero mass; u -> 1 picks the last one
    assert oracle.sample(lg, 0.0) == 0
    spiky = np.full(256, -1e4)
    spiky[[17, 200]] = 0.0
    assert oracle.sample(spiky, 0.0) == 17
    assert oracle.sample(spiky, np.float32(1 - 2 ** -24)) == 200
    assert oracle.sample(spiky, 0.49) == 17 and oracle.sample(spiky, 0.51) == 200


def test_residual_reading_r1_closed_form():
    """W_res = B_res = 0 => x^(j) = x^(j-1) = x^(0) (App. A.1).

    The closed form below evaluates h^(j) = gate(W_prev x0_{n-d} + W_cur x0_n + B + L)
    directly; under the literal §5.1 reading (x^(j) = W_res h + B_res = 0) layers
    >= 2 would see x = 0 instead and this would fail."""
    cfg = synth.Config(3, 4, 6, 16, (1, 4, 2))
    w = synth.make_weights(cfg, 7) * np.float32(3)
    P = synth.split_weights(cfg, w)
    for j in range(3):
        P[f"W_res.{j}"][:] = 0
        P[f"B_res.{j}"][:] = 0
    N, hop = 30, 5
    cond = synth.make_cond(cfg, synth.n_frames_for(N, hop), 3)
    codes = synth.make_codes(N, 3, 16)
    _, lg, _ = run_tf(cfg, w, cond, hop, codes)
    Pd = {k: v.astype(np.float64) for k, v in P.items()}
    hist = np.concatenate([[8, 8], codes.astype(int)])
    x0 = lambda t: (np.zeros(4) if t < 0 else
                    Pd["W_emb_prev"][:, hist[t]] + Pd["W_emb_cur"][:, hist[t + 1]] + Pd["B_emb"])
    for n in range(N):
        q = Pd["B_skip"].copy()
        for j, d in enumerate((1, 4, 2)):
            a = (Pd[f"W_prev.{j}"] @ x0(n - d) + Pd[f"W_cur.{j}"] @ x0(n) + Pd[f"B.{j}"]
                 + cond[n // hop, j].astype(np.float64))
            h = np.tanh(a[:4]) / (1 + np.exp(-a[4:]))
            q += Pd[f"W_skip.{j}"] @ h
        za = np.maximum(Pd["W_relu"] @ np.maximum(q, 0) + Pd["B_relu"], 0)
        np.testing.assert_allclose(lg[n], Pd["W_out"] @ za + Pd["B_out"], rtol=0, atol=1e-13)


def test_determinism():
    cfg = synth.C1
    w = synth.make_weights(cfg, 0)
    N = 200
    cond = synth.make_cond(cfg, synth.n_frames_for(N, 64), 0)
    u = synth.make_uniforms(N, 0)
    a = oracle.run(20, 64, 128, w, cond, 64, N, uniforms=u)
    b = oracle.run(20, 64, 128, w, cond, 64, N, uniforms=u)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_argument_validation():
    cfg = synth.Config(2, 4, 4)
    w = synth.make_weights(cfg, 0)
    cond = synth.make_cond(cfg, 2, 0)
    with pytest.raises(ValueError):  # n_frames too small for N at this hop
        oracle.run(2, 4, 4, w, cond, 4, 20, uniforms=synth.make_uniforms(20))
    with pytest.raises(ValueError):  # wrong blob length
        oracle.run(2, 4, 4, w[:-1], cond, 64, 20, uniforms=synth.make_uniforms(20))


# ---------------------------------------------------------------- App. A.4 sampling strategies (row f3)
# PAPER.md:496-516; readings R24-R27 fix what the paper leaves open.
_rng_s = np.random.default_rng(24)


def _draws(l, us, kind, t=1.0, k=1):
    return np.array([oracle.sample_policy(l, u, kind, t, k) for u in us])


def test_sampler_one_hot_is_fixed_under_every_strategy():
    l = np.zeros(256)
    l[42] = 60.0  # p(42) = 1 - 255 e^-60
    us = _rng_s.random(50, dtype=np.float32)
    for kind, t, k in [(0, 1, 1), (1, 0.5, 1), (1, 3.0, 1), (2, 1, 1), (3, 1, 1), (4, 1, 1), (4, 1, 7)]:
        assert np.all(_draws(l, us, kind, t, k) == 42), (kind, t, k)


def test_temperature_special_cases_pin_the_formula():
    """P^(1/t)/Z: t = 1 is direct sampling; t -> 0 is the mode; t -> inf is uniform."""
    for _ in range(20):
        l = _rng_s.normal(0, 2, 256)
        us = _rng_s.random(20, dtype=np.float32)
        assert np.array_equal(_draws(l, us, 1, 1.0), np.array([oracle.sample(l, u) for u in us]))
        assert np.all(_draws(l, us, 1, 1e-4) == int(np.argmax(l)))
    grid = ((np.arange(256) + 0.5) / 256).astype(np.float32)
    assert np.array_equal(_draws(_rng_s.normal(0, 2, 256), grid, 1, 1e12), np.arange(256))


def test_mode_is_argmax_lowest_index():
    l = _rng_s.normal(0, 1, 256)
    assert oracle.sample_policy(l, 0.9, 3) == int(np.argmax(l))
    l[[17, 99, 200]] = l.max() + 1.0  # three-way tie
    assert oracle.sample_policy(l, 0.1, 3) == 17
    assert oracle.sample_policy(np.zeros(256), 0.5, 3) == 0


def test_mean_rounds_the_expectation():
    assert oracle.sample_policy(np.zeros(256), 0.3, 2) == 128  # E = 127.5 -> 128
    l = np.zeros(256)
    l[[10, 20]] = 80.0
    assert oracle.sample_policy(l, 0.3, 2) == 15
    l = np.zeros(256)
    l[[10, 21]] = 80.0
    assert oracle.sample_policy(l, 0.3, 2) == 16  # 15.5 rounds up
    l = np.zeros(256)
    l[[0, 3]] = [80.0, 80.0 + np.log(3.0)]  # E = (0 + 3 * 3) / 4 = 2.25
    assert oracle.sample_policy(l, 0.3, 2) == 2


def test_top_k_special_cases_and_support():
    for _ in range(20):
        l = _rng_s.normal(0, 2, 256)
        us = _rng_s.random(20, dtype=np.float32)
        assert np.array_equal(_draws(l, us, 4, 1, 256), np.array([oracle.sample(l, u) for u in us]))
        assert np.all(_draws(l, us, 4, 1, 1) == int(np.argmax(l)))
    l = _rng_s.normal(0, 1, 256)
    top5 = set(np.argsort(-l, kind="stable")[:5].tolist())
    grid = ((np.arange(4096) + 0.5) / 4096).astype(np.float32)
    d = _draws(l, grid, 4, 1, 5)
    assert set(d.tolist()) <= top5
    # frequencies over a uniform u grid = the renormalised top-5 distribution (inverse CDF)
    p = np.exp(l - l.max())
    for kk in top5:
        assert abs(np.mean(d == kk) - p[kk] / sum(p[j] for j in top5)) <= 2.0 / 4096
    l2 = np.zeros(256)
    l2[[5, 9, 30]] = 3.0  # ties at the cut: k = 2 keeps the two lower indices
    assert set(_draws(l2, grid[::64], 4, 1, 2).tolist()) == {5, 9}


def test_sampler_rejects_bad_parameters():
    l = np.zeros(256)
    assert oracle.sample_policy(l, 0.5, 1, 0.0) == -1
    assert oracle.sample_policy(l, 0.5, 1, -1.0) == -1
    assert oracle.sample_policy(l, 0.5, 4, 1.0, 0) == -1
    assert oracle.sample_policy(l, 0.5, 4, 1.0, 257) == -1
    assert oracle.sample_policy(l, 0.5, 7) == -1


def test_run_with_strategies_zero_weights_closed_form():
    """All-zero weights give all-zero logits: mode -> 0, mean -> 128 every step; direct and
    temperature draw floor(256 u) (uniform distribution); top-k (k = 256) likewise."""
    cfg = synth.C1
    w = np.zeros(synth.weights_numel(cfg), np.float32)
    N = 64
    cond = synth.make_cond(cfg, synth.n_frames_for(N, 64), 0)
    u = synth.make_uniforms(N, 5)
    floor256 = np.floor(256 * u.astype(np.float64)).astype(np.uint8)
    for sampler, expect in [((3, 1.0, 1), np.zeros(N, np.uint8)), ((2, 1.0, 1), np.full(N, 128, np.uint8)),
                            ((1, 0.7, 1), floor256), ((4, 1.0, 256), floor256)]:
        codes, _, _ = oracle.run(cfg.n_layers, cfg.residual, cfg.skip, w, cond, 64, N, uniforms=u,
                                 sampler=sampler, want_logits=False)
        assert np.array_equal(codes, expect), sampler
