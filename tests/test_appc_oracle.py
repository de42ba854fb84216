"""Pins for the oracle's App. C mode (row f4, DVW_PRECISION_APPC; reading R31).

The paper prints the maximum absolute error of each approximation ("1.5e-3
for tanh, 2.5e-3 for sigmoid, and 2.4e-5 for e^x"; "maximum error 2.4e-5 for
x in (-inf, 0]").  Measured over dense grids, the oracle's functions reproduce those
figures to their printed second digit (tanh 1.514e-3, sigma 2.587e-3, e^x 2.392e-5 where
the fraction does not carry) -- a wrong coefficient, a dropped term or a swapped branch
moves them well outside.  The network-level wiring (every gate and every softmax exp) is
pinned by the independent brute-force oracle's own App. C implementation.
"""
import numpy as np
import pytest

import oracle
from oracle import bruteforce
from paper_1702_07825_b200 import synth

tanh_a = np.vectorize(oracle.appc_tanh)
sig_a = np.vectorize(oracle.appc_sigmoid)
exp_a = np.vectorize(oracle.appc_exp)


def test_appc_tanh_max_error_is_the_papers():
    x = np.linspace(-20.0, 20.0, 400001)
    err = np.abs(tanh_a(x) - np.tanh(x)).max()
    assert 1.4e-3 <= err <= 1.6e-3, err  # printed: 1.5e-3


def test_appc_sigmoid_max_error_is_the_papers():
    x = np.linspace(-20.0, 20.0, 400001)
    err = np.abs(sig_a(x) - 1.0 / (1.0 + np.exp(-x))).max()
    assert 2.4e-3 <= err <= 2.6e-3, err  # printed: 2.5e-3


def test_appc_exp_max_error_is_the_papers():
    """max error 2.4e-5 on (-inf, 0].  The bit-pattern construction doubles it
    where z + g(z) carries out of the fraction (z -> 1; reading R31): there the bound is 2x."""
    x = -np.concatenate([np.logspace(-9, 0, 60001), np.linspace(1.0, 80.0, 120001)])
    e = exp_a(x)
    err = np.abs(e - np.exp(x))
    xl = x / np.log(2.0)
    z = xl - np.floor(xl)
    g = -4.7259162 + 27.7280233 / (4.84252568 - z) - 1.49012907 * z
    carry = z + g >= 2.0
    assert carry.any() and (~carry).any()
    assert 2.3e-5 <= err[~carry].max() <= 2.5e-5, err[~carry].max()
    assert err[carry].max() <= 2 * 2.4e-5 + 1e-6, err[carry].max()


def test_appc_special_values_and_symmetries():
    x = np.linspace(-9.0, 9.0, 3601)
    assert oracle.appc_tanh(0.0) == 0.0 and oracle.appc_sigmoid(0.0) == 0.5
    np.testing.assert_array_equal(tanh_a(-x), -tanh_a(x))              # odd
    np.testing.assert_allclose(sig_a(x) + sig_a(-x), 1.0, atol=1e-15)   # sigma(-x) = 1 - sigma(x)
    assert np.all(np.abs(tanh_a(x)) < 1.0) and np.all((sig_a(x) > 0) & (sig_a(x) < 1))
    # e~ grows like 0.143 x^4 (a polynomial, not exponential, tail): 1 - tanh ~ 2 / e~^2,
    # sigma(-x) ~ 1 / e~
    assert abs(oracle.appc_tanh(60.0) - 1.0) < 1e-12
    assert abs(oracle.appc_sigmoid(-60.0) * (0.143 * 60.0 ** 4) - 1.0) < 1e-2
    # e^x: representable range only; within 2x the printed bound of exp at a few points
    assert oracle.appc_exp(-1000.0) == 0.0 and oracle.appc_exp(-87.0) > 0.0
    for v in (0.0, -0.5, -1.0, -3.3, -10.0):
        assert abs(oracle.appc_exp(v) - np.exp(v)) <= 4.8e-5 * max(np.exp(v), 1e-30) + 1e-12


def tiny(L, r, s, a=16, dil=None, seed=0, scale=1.0):
    cfg = synth.Config(L, r, s, a, tuple(dil) if dil else None)
    return cfg, (synth.make_weights(cfg, seed) * np.float32(scale)).astype(np.float32)


@pytest.mark.parametrize("seed", range(6))
def test_appc_ring_oracle_equals_bruteforce_teacher_forced(seed):
    dil = [[3], [5, 5], [3, 1], [1, 2, 4], [2, 1, 3, 7], [1]][seed]
    cfg, w = tiny(len(dil), 4, 6, a=16, dil=dil, seed=seed, scale=3.0)
    N, hop = 200, [1, 3, 16][seed % 3]
    cond = synth.make_cond(cfg, synth.n_frames_for(N, hop), seed)
    codes = synth.make_codes(N, seed, cfg.levels)
    _, lg, _ = oracle.run(cfg.n_layers, 4, 6, w, cond, hop, N, forced=codes, levels=16, dilations=dil,
                          nonlin="appc")
    _, ex, _ = oracle.run(cfg.n_layers, 4, 6, w, cond, hop, N, forced=codes, levels=16, dilations=dil)
    bf = bruteforce.forward_logits(w, cfg.n_layers, 4, 6, codes, cond, hop, 16, dil, nonlin="appc")
    assert np.max(np.abs(lg - bf)) <= 1e-12
    d = np.max(np.abs(lg - ex))
    assert 1e-5 < d < 0.5, d  # the approximations are in the gates, and they are small


@pytest.mark.parametrize("seed", range(3))
def test_appc_ring_oracle_equals_bruteforce_free_running(seed):
    dil = [[1, 2, 4], [5, 5], [3, 1]][seed]
    cfg, w = tiny(len(dil), 4, 6, a=16, dil=dil, seed=seed, scale=4.0)
    N, hop = 64, 8
    cond = synth.make_cond(cfg, synth.n_frames_for(N, hop), seed)
    u = synth.make_uniforms(N, seed)
    codes, _, _ = oracle.run(cfg.n_layers, 4, 6, w, cond, hop, N, uniforms=u, levels=16, dilations=dil,
                             nonlin="appc")
    bf = bruteforce.generate(w, cfg.n_layers, 4, 6, cond, hop, u, N, 16, dil, nonlin="appc")
    assert np.array_equal(codes, bf)
    assert len(set(codes.tolist())) >= 4  # not a constant trajectory


def test_appc_zero_weights_still_floor_256u():
    """Equal logits => every e_k = appc_exp(0), the same number => p uniform => y = floor(256 u)."""
    cfg = synth.C1
    w = np.zeros(synth.weights_numel(cfg), np.float32)
    N, hop = 300, 64
    cond = synth.make_cond(cfg, synth.n_frames_for(N, hop), 0) * 0
    u = synth.make_uniforms(N, 0)
    codes, _, _ = oracle.run(cfg.n_layers, cfg.residual, cfg.skip, w, cond, hop, N, uniforms=u, nonlin="appc")
    np.testing.assert_array_equal(codes, np.floor(u.astype(np.float64) * 256).astype(np.uint8))


def test_appc_rejects_unknown_mode():
    cfg, w = tiny(1, 4, 6)
    cond = synth.make_cond(cfg, 4, 0)
    with pytest.raises(KeyError):
        oracle.run(1, 4, 6, w, cond, 1, 4, uniforms=synth.make_uniforms(4, 0), levels=16, nonlin="fast")
