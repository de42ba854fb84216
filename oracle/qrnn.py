"""Plain fp64 NumPy oracle of the conditioning network (App. A.2) --
TEST INFRASTRUCTURE: only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import it; the product path never does.

A unidirectional QRNN layer with fo-pooling and 2x1 convolutions:
    h~_t = tanh(W_h * x + B_h),  o_t = sigma(W_o * x + B_o),  f_t = sigma(W_f * x + B_f)
    h_t  = f_t h_{t-1} + (1 - f_t) h~_t,   z_t = o_t h_t,   h_0 = 0
where "W * x" is the 2x1 convolution over time W[0] x_{t-1} + W[1] x_t (x_{-1} = 0).  The
bidirectional layer runs one QRNN on the sequence and one on the reversed sequence and
stacks their channels; two such layers; then the channels are interleaved so
the WaveNet's tanh and sigmoid halves both see forward and backward channels.
Readings (R28-R30): the backward QRNN's taps are x_{t+1}, x_t in original time
(the forward rule applied to the reversed copy); "interleave" means out[2i] = forward channel
i, out[2i+1] = backward channel i of the second layer; each WaveNet layer j then gets its own
linear projection L^(j)_t = P^(j) out_t + B^(j) to 2r channels (SPEC build_conditioning),
at frame rate -- the generator repeats frame f for samples [f hop, (f+1) hop).

Pins (tests/test_qrnn_oracle.py): the fo-pooling recurrence against its unrolled closed form,
the forget-gate limits (f -> 0: h = h~; f -> 1: h carries), zero weights giving exactly the
projection bias, causality of each direction (a frame perturbation moves only frames on its
side), reversal of the input swapping the two directions, shapes / interleave / blob size.
The output VALUES for random weights are "parity unpinned by the paper" (it prints none):
beyond those properties they are pinned only by the GPU conditioner agreeing with them.

Weight blob (fp32, this order), per QRNN layer q = 1, 2 (C_in = features for q = 1, 2H for
q = 2), per direction (forward, then backward):
    W [3 gates: h, o, f][2 taps: t-1, t][H][C_in],  B [3][H]
then P [l][2r][2H], B_P [l][2r].
"""
from __future__ import annotations

import numpy as np


def numel(c_in: int, hidden: int, n_layers: int, residual: int) -> int:
    n = 0
    for cin in (c_in, 2 * hidden):
        n += 2 * (3 * 2 * hidden * cin + 3 * hidden)
    return n + n_layers * 2 * residual * 2 * hidden + n_layers * 2 * residual


def unpack(blob: np.ndarray, c_in: int, hidden: int, n_layers: int, residual: int):
    """Split the blob into fp64 arrays: [(Wf, Bf, Wb, Bb) for each QRNN layer], P, B_P."""
    b = np.asarray(blob, dtype=np.float32).astype(np.float64)
    assert b.size == numel(c_in, hidden, n_layers, residual), (b.size, numel(c_in, hidden, n_layers, residual))
    off = 0

    def take(shape):
        nonlocal off
        n = int(np.prod(shape))
        a = b[off:off + n].reshape(shape)
        off += n
        return a

    layers = []
    for cin in (c_in, 2 * hidden):
        wf, bf = take((3, 2, hidden, cin)), take((3, hidden))
        wb, bb = take((3, 2, hidden, cin)), take((3, hidden))
        layers.append((wf, bf, wb, bb))
    P = take((n_layers, 2 * residual, 2 * hidden))
    BP = take((n_layers, 2 * residual))
    return layers, P, BP


def sigmoid(v):
    return 1.0 / (1.0 + np.exp(-v))


def qrnn_forward(x: np.ndarray, W: np.ndarray, B: np.ndarray) -> np.ndarray:
    """One unidirectional fo-pooling QRNN over x [T][C_in] -> z [T][H],
    step by step in the paper's order."""
    T = x.shape[0]
    H = B.shape[1]
    z = np.zeros((T, H))
    h = np.zeros(H)
    x_prev = np.zeros(x.shape[1])
    for t in range(T):
        conv = [W[g, 0] @ x_prev + W[g, 1] @ x[t] + B[g] for g in range(3)]  # 2x1 convolution
        h_tilde = np.tanh(conv[0])
        o = sigmoid(conv[1])
        f = sigmoid(conv[2])
        h = f * h + (1.0 - f) * h_tilde
        z[t] = o * h
        x_prev = x[t]
    return z


def qrnn_bidirectional(x: np.ndarray, Wf, Bf, Wb, Bb) -> np.ndarray:
    """Forward QRNN on x, backward QRNN on the reversed copy (re-reversed), channels stacked
    [forward | backward]."""
    zf = qrnn_forward(x, Wf, Bf)
    zb = qrnn_forward(x[::-1], Wb, Bb)[::-1]
    return np.concatenate([zf, zb], axis=1)


def interleave(z: np.ndarray) -> np.ndarray:
    """[forward H | backward H] -> channel 2i = forward i, 2i+1 = backward i (reading R29)."""
    H = z.shape[1] // 2
    out = np.empty_like(z)
    out[:, 0::2] = z[:, :H]
    out[:, 1::2] = z[:, H:]
    return out


def condition(features: np.ndarray, blob: np.ndarray, hidden: int, n_layers: int, residual: int) -> np.ndarray:
    """features [T][C_in] -> per-layer conditioning L [T][l][2r] at frame rate."""
    x = np.asarray(features, dtype=np.float32).astype(np.float64)
    layers, P, BP = unpack(blob, x.shape[1], hidden, n_layers, residual)
    for (wf, bf, wb, bb) in layers:
        x = qrnn_bidirectional(x, wf, bf, wb, bb)
    out = interleave(x)
    T = out.shape[0]
    L = np.empty((T, n_layers, 2 * residual))
    for j in range(n_layers):
        L[:, j, :] = out @ P[j].T + BP[j]
    return L
