"""Pins of the conditioning-network oracle (oracle/qrnn.py; App. A.2;
SURVEY.md §8(f) row f2) against closed forms, special cases and invariants."""
import numpy as np
import pytest

from oracle import qrnn

RNG = np.random.default_rng(28)


def rand_layer(cin, H, scale=1.0):
    b = 1.0 / np.sqrt(2 * cin)
    return RNG.uniform(-b, b, (3, 2, H, cin)) * scale, RNG.uniform(-b, b, (3, H)) * scale


def test_fo_pooling_closed_form_unrolled():
    """h_t = sum_{s<=t} (1 - f_s) h~_s prod_{s<u<=t} f_u, brute force over s (no recurrence)."""
    T, C, H = 17, 5, 4
    x = RNG.uniform(-1, 1, (T, C))
    W, B = rand_layer(C, H, 3.0)
    z = qrnn.qrnn_forward(x, W, B)
    xp = np.vstack([np.zeros((1, C)), x[:-1]])
    conv = [np.einsum("hc,tc->th", W[g, 0], xp) + np.einsum("hc,tc->th", W[g, 1], x) + B[g] for g in range(3)]
    ht, o, f = np.tanh(conv[0]), 1 / (1 + np.exp(-conv[1])), 1 / (1 + np.exp(-conv[2]))
    for t in range(T):
        h = np.zeros(H)
        for s in range(t + 1):
            h += (1 - f[s]) * ht[s] * np.prod(f[s + 1:t + 1], axis=0)
        assert np.allclose(z[t], o[t] * h, atol=1e-12, rtol=0)


def test_forget_gate_limits():
    """f = 1 holds h_0 = 0 (z = 0); f = 0 is memoryless, z_t = o_t tanh(W_h * x + B_h) (SPEC)."""
    T, C, H = 12, 6, 3
    x = RNG.uniform(-1, 1, (T, C))
    W, B = rand_layer(C, H)
    B1 = B.copy()
    B1[2] = 60.0
    assert np.max(np.abs(qrnn.qrnn_forward(x, W, B1))) < 1e-20
    B0 = B.copy()
    B0[2] = -60.0
    xp = np.vstack([np.zeros((1, C)), x[:-1]])
    conv_h = xp @ W[0, 0].T + x @ W[0, 1].T + B0[0]
    conv_o = xp @ W[1, 0].T + x @ W[1, 1].T + B0[1]
    assert np.allclose(qrnn.qrnn_forward(x, W, B0), np.tanh(conv_h) / (1 + np.exp(-conv_o)), atol=1e-12)


def test_zero_weights_give_zero_conditioning_plus_bias():
    cin, H, l, r = 7, 4, 3, 8
    blob = np.zeros(qrnn.numel(cin, H, l, r), np.float32)
    x = RNG.uniform(-1, 1, (9, cin))
    assert np.all(qrnn.condition(x, blob, H, l, r) == 0.0)  # h~ = tanh(0) = 0 -> z = 0, P = B = 0


def test_causality_of_each_direction():
    T, C, H = 20, 4, 3
    x = RNG.uniform(-1, 1, (T, C))
    Wf, Bf = rand_layer(C, H, 2.0)
    Wb, Bb = rand_layer(C, H, 2.0)
    z = qrnn.qrnn_bidirectional(x, Wf, Bf, Wb, Bb)
    x2 = x.copy()
    x2[11] += 0.5
    z2 = qrnn.qrnn_bidirectional(x2, Wf, Bf, Wb, Bb)
    assert np.array_equal(z2[:11, :H], z[:11, :H]) and not np.array_equal(z2[11, :H], z[11, :H])
    assert np.array_equal(z2[12:, H:], z[12:, H:]) and not np.array_equal(z2[11, H:], z[11, H:])


def test_reversal_swaps_directions():
    T, C, H = 15, 4, 3
    x = RNG.uniform(-1, 1, (T, C))
    Wf, Bf = rand_layer(C, H, 2.0)
    Wb, Bb = rand_layer(C, H, 2.0)
    z = qrnn.qrnn_bidirectional(x, Wf, Bf, Wb, Bb)
    zr = qrnn.qrnn_bidirectional(x[::-1].copy(), Wb, Bb, Wf, Bf)
    assert np.allclose(zr[::-1][:, :H], z[:, H:], atol=1e-14)
    assert np.allclose(zr[::-1][:, H:], z[:, :H], atol=1e-14)


def test_shapes_lengths_interleave_and_blob():
    cin, H, l, r = 6, 4, 3, 8
    blob = RNG.uniform(-0.3, 0.3, qrnn.numel(cin, H, l, r)).astype(np.float32)
    for T in (1, 2, 13):
        L = qrnn.condition(RNG.uniform(-1, 1, (T, cin)), blob, H, l, r)
        assert L.shape == (T, l, 2 * r)
    assert qrnn.condition(np.zeros((0, cin)), blob, H, l, r).shape == (0, l, 2 * r)
    z = np.arange(12.0).reshape(2, 6)  # [f0 f1 f2 | b0 b1 b2]
    assert np.array_equal(qrnn.interleave(z)[0], [0, 3, 1, 4, 2, 5])
    with pytest.raises(AssertionError):
        qrnn.unpack(blob[:-1], cin, H, l, r)
