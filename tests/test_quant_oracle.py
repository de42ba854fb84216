"""Pins for the weight-quantisation oracle (row f4; reading R32).

The paper states only that weights were quantised to int16 with no audible change; the
scheme (symmetric, per row, fp32 arithmetic) is reading R32.  Pinned here by closed forms:
on-grid matrices are reproduced bit for bit, every element moves by at most half a step,
the largest element of a row maps to +-(2^(bits-1) - 1), zero rows and biases are untouched,
and the roster agrees with the C oracle's independent blob size.
"""
import numpy as np
import pytest

import oracle
from oracle import quant
from paper_1702_07825_b200 import synth


@pytest.mark.parametrize("shape", [(1, 4, 6, 16), (20, 64, 256, 256), (3, 128, 128, 256), (40, 64, 256, 256)])
def test_roster_matches_the_c_oracle_blob(shape):
    L, r, s, a = shape
    mats, numel = quant.roster(L, r, s, a)
    assert numel == oracle.weights_numel(L, r, s, a)
    assert len(mats) == 4 * L + 4
    ends = [off + rows * cols for off, rows, cols in mats]
    assert all(e <= o for e, (o, _, _) in zip(ends, mats[1:]))  # disjoint, in blob order


@pytest.mark.parametrize("bits", [8, 16])
def test_on_grid_matrix_is_reproduced_exactly(bits):
    Q = (1 << (bits - 1)) - 1
    rng = np.random.default_rng(bits)
    k = rng.integers(-Q, Q + 1, size=(9, 33))
    k[:, 0] = np.where(rng.random(9) < 0.5, Q, -Q)  # each row reaches the full range
    W = (k * 2.0 ** -10).astype(np.float32)
    np.testing.assert_array_equal(quant.quantize_rows(W, bits), W)
    q, sc = quant.quantize_codes(W, bits)
    np.testing.assert_array_equal(q, k)
    assert np.all(sc == np.float32(2.0 ** -10))


@pytest.mark.parametrize("bits", [8, 16])
def test_half_step_bound_codes_range_and_extremes(bits):
    Q = (1 << (bits - 1)) - 1
    rng = np.random.default_rng(7)
    W = (rng.standard_normal((64, 200)) * rng.uniform(0.01, 3.0, (64, 1))).astype(np.float32)
    Wq = quant.quantize_rows(W, bits)
    q, sc = quant.quantize_codes(W, bits)
    assert np.all(np.abs(q) <= Q)
    amax = np.argmax(np.abs(W), axis=1)
    assert np.all(np.abs(q[np.arange(64), amax]) == Q)
    step = sc[:, None].astype(np.float64)
    err = np.abs(Wq.astype(np.float64) - W.astype(np.float64))
    assert np.all(err <= 0.5 * step * (1 + 2 ** -20) + np.abs(W) * 2 ** -23)
    assert np.all(np.sign(Wq) * np.sign(W) >= 0)  # never flips a sign
    # the codes are a fixed point of the scheme
    q2, _ = quant.quantize_codes(Wq, bits)
    np.testing.assert_array_equal(q2, q)


def test_zero_rows_and_biases_untouched():
    cfg = synth.Config(2, 8, 16, 256)
    w = synth.make_weights(cfg, 3)
    mats, numel = quant.roster(cfg.n_layers, 8, 16, 256)
    off, rows, cols = mats[2]  # layer 0's W_res: zero one row
    w[off + cols:off + 2 * cols] = 0.0
    wq = quant.quantize_weights(w, cfg.n_layers, 8, 16, 16)
    assert np.all(wq[off + cols:off + 2 * cols] == 0.0)
    in_mat = np.zeros(numel, bool)
    for o, r_, c_ in mats:
        in_mat[o:o + r_ * c_] = True
    np.testing.assert_array_equal(wq[~in_mat], w[~in_mat])
    assert not np.array_equal(wq[in_mat], w[in_mat])


def test_int16_keeps_logits_within_the_gate_and_int8_is_coarser():
    """PAPER.md:385 'no change in perceptual quality' at int16: teacher-forced logits move by
    far less than the north_star 1e-3 gate; int8 moves them more."""
    cfg = synth.C1
    N, hop = 200, 64
    w = synth.make_weights(cfg, 0)
    cond = synth.make_cond(cfg, synth.n_frames_for(N, hop), 0)
    codes = synth.make_codes(N, 0)
    run = lambda blob: oracle.run(cfg.n_layers, cfg.residual, cfg.skip, blob, cond, hop, N, forced=codes)[1]
    base = run(w)
    d16 = np.max(np.abs(run(quant.quantize_weights(w, cfg.n_layers, cfg.residual, cfg.skip, 16)) - base))
    d8 = np.max(np.abs(run(quant.quantize_weights(w, cfg.n_layers, cfg.residual, cfg.skip, 8)) - base))
    print(f"teacher-forced max|dlogit| int16 {d16:.2e}, int8 {d8:.2e}")
    assert 0 < d16 < 1e-3 and d16 < d8 / 50


# ---- reading R33: per-tensor scheme (SPEC.md quantize_weights examples)
def test_per_tensor_spec_examples():
    q, sc = quant.quantize_tensor_codes(np.array([[0.0, 1.0, -1.0]], dtype=np.float32), 16)
    np.testing.assert_array_equal(q, [[0, 32767, -32767]])
    assert sc == np.float32(1.0 / 32767)
    qz, scz = quant.quantize_tensor_codes(np.zeros((3, 5), dtype=np.float32), 16)
    assert np.all(qz == 0) and scz == np.float32(1.0)
    np.testing.assert_array_equal(quant.quantize_tensor(np.zeros((3, 5), np.float32), 16), 0.0)


@pytest.mark.parametrize("bits", [8, 16])
def test_per_tensor_half_step_bound_and_single_scale(bits):
    cfg = synth.Config(2, 64, 128)
    w = synth.make_weights(cfg, 7)
    wq = quant.quantize_weights(w, cfg.n_layers, cfg.residual, cfg.skip, bits, scheme="per_tensor")
    mats, _ = quant.roster(cfg.n_layers, cfg.residual, cfg.skip)
    Q = (1 << (bits - 1)) - 1
    for off, rows, cols in mats:
        W = w[off:off + rows * cols].reshape(rows, cols)
        Wq = wq[off:off + rows * cols].reshape(rows, cols)
        q, sc = quant.quantize_tensor_codes(W, bits)
        assert np.max(np.abs(q)) == Q                      # the largest element reaches the end code
        # SPEC's bound s/2, plus the fp32 rounding of the quotient W/s and of the product q s
        # (each <= 2^-24 |W| relative)
        assert np.all(np.abs(Wq.astype(np.float64) - W) <= np.float64(sc) / 2 + np.abs(W) * 2.0 ** -22)
        np.testing.assert_array_equal(Wq, (q * np.float64(sc)).astype(np.float32))
    # per-tensor is coarser than per-row: it differs from the per-row blob on some matrix
    wr = quant.quantize_weights(w, cfg.n_layers, cfg.residual, cfg.skip, bits)
    assert not np.array_equal(wq, wr)
    # biases untouched
    mask = np.ones(w.size, bool)
    for off, rows, cols in mats:
        mask[off:off + rows * cols] = False
    np.testing.assert_array_equal(wq[mask], w[mask])
