"""Second, independent fp64 oracle: the WaveNet variant as a dilated causal
convolution network evaluated over the whole history, with no ring buffers.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Tiny models only.

It follows App. A.1 literally:
  x^(0) = W_embed * y + B_embed        -- a 2x1 convolution over the one-hot codes
                                        (PAPER.md:431); taps are the codes of the two
                                        previous timesteps (reading R3), codes at
                                        negative times are a/2 (reading R4)
  h'^(i)_t = W_prev x^(i-1)_{t-d} + W_cur x^(i-1)_t + B^(i) + L^(i)_t
             with zero left-padding x^(i-1)_{t<0} = 0 (reading R4)
  h^(i) = tanh(h'_{0:r}) * sigma(h'_{r:2r})
  x^(i) = x^(i-1) + W_r h^(i) + B_r
  z_s = relu(W_skip [h^(1); ...; h^(l)] + B_skip)
  z_a = relu(W_relu z_s + B_relu); p = softmax(W_out z_a + B_out)
The skip projection is done as ONE s x (l r) matrix on the concatenated h,
as App. A.1 writes it (the ring oracle sums per-layer blocks, §5.1 step 2d).
Upsampling by repetition: L_t = cond[t // hop].
"""
from __future__ import annotations

from typing import Optional, Sequence

import numpy as np


def _split(blob: np.ndarray, L: int, r: int, s: int, a: int) -> dict:
    w = np.asarray(blob, dtype=np.float64)
    out, off = {}, 0

    def take(name, shape):
        nonlocal off
        n = int(np.prod(shape))
        out[name] = w[off:off + n].reshape(shape)
        off += n

    for j in range(L):
        take(("W_prev", j), (2 * r, r))
        take(("W_cur", j), (2 * r, r))
        take(("B", j), (2 * r,))
        take(("W_res", j), (r, r))
        take(("B_res", j), (r,))
        take(("W_skip", j), (s, r))
    for name, shape in (("W_emb_prev", (r, a)), ("W_emb_cur", (r, a)), ("B_emb", (r,)),
                        ("B_skip", (s,)), ("W_relu", (a, s)), ("B_relu", (a,)),
                        ("W_out", (a, a)), ("B_out", (a,))):
        take(name, shape)
    assert off == w.size, (off, w.size)
    return out


# App. C's approximations, vectorised independently of dvw_oracle.c.
def _etilde(x):
    return 1.0 + np.abs(x) + 0.5658 * x ** 2 + 0.143 * x ** 4


def _tanh_appc(x):
    e = _etilde(x)
    return np.sign(x) * (e - 1.0 / e) / (e + 1.0 / e)


def _sigmoid_appc(x):
    e = _etilde(x)
    return np.where(x >= 0.0, e / (1.0 + e), 1.0 / (1.0 + e))


def _exp_appc(x):
    """2^(x/ln2) through the fp32 bit pattern (x + 126 + g(z)) 2^23."""
    xl = np.asarray(x, dtype=np.float64) / np.log(2.0)
    z = xl - np.floor(xl)
    g = -4.7259162 + 27.7280233 / (4.84252568 - z) - 1.49012907 * z
    ok = xl >= -126.0
    bits = np.trunc(np.where(ok, (xl + 126.0 + g) * 2.0 ** 23, 0.0)).astype(np.int32)
    return np.where(ok, bits.view(np.float32).astype(np.float64), 0.0)


def forward_logits(blob, L: int, r: int, s: int, codes_in: np.ndarray, cond: np.ndarray,
                   hop: int, a: int = 256, dilations: Optional[Sequence[int]] = None,
                   nonlin: str = "exact") -> np.ndarray:
    """Logits for t = 0..T-1 given the code history.

    ``codes_in[t]`` is the code emitted at step t (only t < T-1 matter for the
    logits at T-1).  Returns float64 [T][a].
    """
    P = _split(blob, L, r, s, a)
    d = list(dilations) if dilations is not None else [1 << (j % 10) for j in range(L)]
    T = len(codes_in)
    hist = np.concatenate([[a // 2, a // 2], np.asarray(codes_in, dtype=np.int64)])
    # y_{t-2} = hist[t], y_{t-1} = hist[t+1]
    x = P["W_emb_prev"][:, hist[0:T]].T + P["W_emb_cur"][:, hist[1:T + 1]].T + P["B_emb"]
    c = np.asarray(cond, dtype=np.float64)
    frames = np.arange(T) // hop
    hs = []
    for j in range(L):
        xs = np.zeros_like(x)
        if d[j] < T:
            xs[d[j]:] = x[:T - d[j]]
        hp = xs @ P[("W_prev", j)].T + x @ P[("W_cur", j)].T + P[("B", j)] + c[frames, j, :]
        if nonlin == "appc":
            h = _tanh_appc(hp[:, :r]) * _sigmoid_appc(hp[:, r:])
        else:
            h = np.tanh(hp[:, :r]) * (1.0 / (1.0 + np.exp(-hp[:, r:])))
        x = x + h @ P[("W_res", j)].T + P[("B_res", j)]
        hs.append(h)
    Hcat = np.concatenate(hs, axis=1)  # [T][l r], layer-major like App. A.1's stacked h
    Wskip = np.concatenate([P[("W_skip", j)] for j in range(L)], axis=1)  # s x (l r)
    zs = np.maximum(Hcat @ Wskip.T + P["B_skip"], 0.0)
    za = np.maximum(zs @ P["W_relu"].T + P["B_relu"], 0.0)
    return za @ P["W_out"].T + P["B_out"]


def draw(logits: np.ndarray, u: float, nonlin: str = "exact") -> int:
    """Inverse-CDF draw (reading R11) written with numpy primitives."""
    l = np.asarray(logits, dtype=np.float64)
    e = _exp_appc(l - l.max()) if nonlin == "appc" else np.exp(l - l.max())
    cdf = np.cumsum(e)
    k = int(np.searchsorted(cdf, float(np.float32(u)) * cdf[-1], side="right"))
    if k >= l.size:
        k = int(np.nonzero(e > 0)[0][-1])
    return k


def generate(blob, L: int, r: int, s: int, cond: np.ndarray, hop: int, uniforms: np.ndarray,
             n_samples: int, a: int = 256, dilations=None, nonlin: str = "exact") -> np.ndarray:
    """Free-running generation by full recomputation at every step (O(N^2))."""
    codes = np.zeros(n_samples, dtype=np.int64)
    for n in range(n_samples):
        lg = forward_logits(blob, L, r, s, codes[:n + 1], cond, hop, a, dilations, nonlin)[n]
        codes[n] = draw(lg, uniforms[n], nonlin)
    return codes.astype(np.uint8)
