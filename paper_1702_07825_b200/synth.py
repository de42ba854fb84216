"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This module holds NONE of the method's arithmetic: it only draws random numbers
and lays them out in the boundary's documented order (include/dvw.h).  It is
the one module both sides may use.

Recipe ("Synthetic inputs"):

* weights: ``np.random.default_rng(seed)`` (PCG64), uniform(+-1/sqrt(fan_in)),
  drawn in fp64 tensor by tensor in blob order, rounded to fp32.
  fan_in = r for W_prev, W_cur, B, W_res, B_res; l*r for W_skip, B_skip;
  s for W_relu, B_relu; a for W_out, B_out, W_emb_prev, W_emb_cur, B_emb.
  Profile "peaky" multiplies W_out and B_out by 30 (logit std ~0.05 -> ~1.4).
* conditioning for utterance u: ``default_rng([1, u]).uniform(-0.5, 0.5,
  (n_frames, l, 2r))`` as fp32, one frame per ``hop`` = 64 samples
  (App. A.3: 256 Hz features, 16,384 Hz audio).
* uniforms for utterance u: ``default_rng([2, u]).random(N, dtype=float32)``.

Keying every input by (role, u) makes it independent of batch composition and
GPU count (SURVEY.md §8(e) sharding invariance).
"""
from __future__ import annotations

import dataclasses
import math
from typing import List, Optional, Sequence, Tuple

import numpy as np

LEVELS = 256  # a: mu-law levels (§3.4; App. A.1)
DEFAULT_HOP = 64  # 16,384 Hz / 256 Hz (App. A.3)
AUDIO_HZ = 16000  # BASELINE.json real-time rate


@dataclasses.dataclass(frozen=True)
class Config:
    """WaveNet size (§3.4: l layers, r residual, s skip, a levels)."""

    n_layers: int
    residual: int
    skip: int
    levels: int = LEVELS
    dilations: Optional[Tuple[int, ...]] = None  # None -> 2^((j-1) mod 10)

    def dilation_list(self) -> List[int]:
        if self.dilations is not None:
            assert len(self.dilations) == self.n_layers
            return list(self.dilations)
        return [2 ** (j % 10) for j in range(self.n_layers)]


# The BASELINE.json configs (SURVEY.md §8(a) shorthand).
C1 = Config(20, 64, 128)
C2 = Config(20, 64, 256)
C3 = Config(40, 64, 256)
C4 = Config(20, 128, 256)
C5 = Config(40, 64, 256)


def roster(cfg: Config) -> List[Tuple[str, Tuple[int, ...], int]]:
    """(name, shape, fan_in) in blob order (include/dvw.h "Weight blob")."""
    L, r, s, a = cfg.n_layers, cfg.residual, cfg.skip, cfg.levels
    out = []
    for j in range(L):
        out += [
            (f"W_prev.{j}", (2 * r, r), r),
            (f"W_cur.{j}", (2 * r, r), r),
            (f"B.{j}", (2 * r,), r),
            (f"W_res.{j}", (r, r), r),
            (f"B_res.{j}", (r,), r),
            (f"W_skip.{j}", (s, r), L * r),
        ]
    out += [
        ("W_emb_prev", (r, a), a),
        ("W_emb_cur", (r, a), a),
        ("B_emb", (r,), a),
        ("B_skip", (s,), L * r),
        ("W_relu", (a, s), s),
        ("B_relu", (a,), s),
        ("W_out", (a, a), a),
        ("B_out", (a,), a),
    ]
    return out


def weights_numel(cfg: Config) -> int:
    return int(sum(int(np.prod(shape)) for _, shape, _ in roster(cfg)))


def make_weights(cfg: Config, seed: int = 0, profile: str = "default") -> np.ndarray:
    """Flat fp32 blob in roster order."""
    rng = np.random.default_rng(seed)
    parts = []
    for name, shape, fan_in in roster(cfg):
        bound = 1.0 / math.sqrt(fan_in)
        t = rng.uniform(-bound, bound, size=shape)  # fp64 draw
        if profile == "peaky" and name in ("W_out", "B_out"):
            t = t * 30.0
        elif profile not in ("default", "peaky"):
            raise ValueError(f"unknown weight profile {profile!r}")
        parts.append(t.astype(np.float32).ravel())
    return np.concatenate(parts)


def split_weights(cfg: Config, blob: np.ndarray) -> dict:
    """Views of the blob by roster name (layout bookkeeping only)."""
    out, off = {}, 0
    for name, shape, _ in roster(cfg):
        n = int(np.prod(shape))
        out[name] = blob[off:off + n].reshape(shape)
        off += n
    assert off == blob.size
    return out


def n_frames_for(n_samples: int, hop: int) -> int:
    return max(1, -(-n_samples // hop))


def make_cond(cfg: Config, n_frames: int, utt: int = 0) -> np.ndarray:
    """fp32 [n_frames][l][2r] frame-rate conditioning for utterance ``utt``."""
    rng = np.random.default_rng([1, utt])
    return rng.uniform(-0.5, 0.5, (n_frames, cfg.n_layers, 2 * cfg.residual)).astype(np.float32)


def make_uniforms(n_samples: int, utt: int = 0) -> np.ndarray:
    """fp32 [N] in [0, 1), 24-bit granularity."""
    rng = np.random.default_rng([2, utt])
    return rng.random(n_samples, dtype=np.float32)


def make_batch(cfg: Config, n_samples: int, utts: Sequence[int], hop: int = DEFAULT_HOP):
    """Stacked (cond [U][F][l][2r], uniforms [U][N]) for a list of utterance ids."""
    nf = n_frames_for(n_samples, hop)
    cond = np.stack([make_cond(cfg, nf, u) for u in utts])
    uni = np.stack([make_uniforms(n_samples, u) for u in utts])
    return cond, uni


# ---------------------------------------------------------------- counter-based inputs (batched)
# The batched workloads (C4: 256 x 5 s, C5: 2,048 x 5 s -- 52 GB of conditioning) are drawn on
# the device.  Each element is a stateless hash of (role, utterance, element index), so an
# utterance's inputs never depend on which other utterances share its batch, its rank or the
# GPU count (sharding invariance), and numpy (host) and torch (device)
# produce the same fp32 values.  Hash: Wellons' "lowbias32" 32-bit integer permutation,
# chained over the key; value = top 24 bits / 2^24 (exact in fp32), in [0, 1).
_M32 = 0xFFFFFFFF
ROLE_COND, ROLE_UNIFORM = 1, 2


def _mix32_np(x):
    x = np.asarray(x, dtype=np.uint64) & _M32
    x ^= x >> np.uint64(16)
    x = (x * np.uint64(0x7FEB352D)) & _M32
    x ^= x >> np.uint64(15)
    x = (x * np.uint64(0x846CA68B)) & _M32
    x ^= x >> np.uint64(16)
    return x


def _keys(role: int, utt: int):
    k0 = int(_mix32_np((role * 0x9E3779B9 + 0x632BE5AB) & _M32))
    k1 = int(_mix32_np(k0 ^ (utt & _M32)))
    return k0, k1


def hashed_uniform_np(role: int, utt: int, idx) -> np.ndarray:
    """fp32 U[0, 1) of element(s) idx of (role, utterance) -- host reference of the device draw."""
    k0, k1 = _keys(role, utt)
    v = _mix32_np(_mix32_np(np.asarray(idx, dtype=np.uint64) ^ np.uint64(k1)) ^ np.uint64(k0))
    return ((v >> np.uint64(8)).astype(np.float64) * 2.0 ** -24).astype(np.float32)


def make_cond_hashed(cfg: Config, n_frames: int, utt: int) -> np.ndarray:
    """Host copy of utterance utt's hashed conditioning: U(-0.5, 0.5) fp32 [F][l][2r]."""
    n = n_frames * cfg.n_layers * 2 * cfg.residual
    v = hashed_uniform_np(ROLE_COND, utt, np.arange(n, dtype=np.uint64)) - np.float32(0.5)
    return v.reshape(n_frames, cfg.n_layers, 2 * cfg.residual)


def make_uniforms_hashed(n_samples: int, utt: int) -> np.ndarray:
    return hashed_uniform_np(ROLE_UNIFORM, utt, np.arange(n_samples, dtype=np.uint64))


def _mix32_torch(x):
    # int64 holding a uint32; products wrap mod 2^64 and the mask keeps the exact low 32 bits
    x = x ^ (x >> 16)
    x = (x * 0x7FEB352D) & _M32
    x = x ^ (x >> 15)
    x = (x * 0x846CA68B) & _M32
    return x ^ (x >> 16)


def _hashed_fill_torch(out, role: int, utts, chunk_elems: int = 1 << 27):
    """out [U][...] float32 (any device) <- hashed U[0, 1) per (role, utts[i], flat index)."""
    import torch
    per = out[0].numel() if out.shape[0] else 0
    flat = out.view(out.shape[0], -1)
    step = max(1, chunk_elems // max(per, 1))
    idx = torch.arange(per, dtype=torch.int64, device=out.device)
    for i0 in range(0, out.shape[0], step):
        us = utts[i0:i0 + step]
        ks = [_keys(role, int(u)) for u in us]
        k0 = torch.tensor([k[0] for k in ks], dtype=torch.int64, device=out.device)[:, None]
        k1 = torch.tensor([k[1] for k in ks], dtype=torch.int64, device=out.device)[:, None]
        v = _mix32_torch(_mix32_torch(idx[None, :] ^ k1) ^ k0)
        flat[i0:i0 + len(us)] = ((v >> 8).to(torch.float64) * 2.0 ** -24).to(torch.float32)


def make_batch_hashed_torch(cfg: Config, n_samples: int, utts: Sequence[int], hop: int, device):
    """(cond [U][F][l][2r], uniforms [U][N]) for utterance ids `utts`, drawn on `device` with
    the counter-based hash: equal to make_cond_hashed / make_uniforms_hashed element for element."""
    import torch
    nf = n_frames_for(n_samples, hop)
    cond = torch.empty((len(utts), nf, cfg.n_layers, 2 * cfg.residual), dtype=torch.float32, device=device)
    uni = torch.empty((len(utts), n_samples), dtype=torch.float32, device=device)
    _hashed_fill_torch(cond, ROLE_COND, list(utts))
    cond -= 0.5
    _hashed_fill_torch(uni, ROLE_UNIFORM, list(utts))
    return cond, uni


def make_codes(n_samples: int, utt: int = 0, levels: int = LEVELS) -> np.ndarray:
    """Random uint8 code history for teacher-forced runs (role key 3)."""
    rng = np.random.default_rng([3, utt])
    return rng.integers(0, levels, n_samples, dtype=np.int64).astype(np.uint8)


# ---------------------------------------------------------------- conditioning network (row f2)
# Features: 227 channels per 256 Hz frame (one-hot phoneme with two previous and two next
# phonemes, voiced flag, normalised log F0 -- PAPER.md:485-489 App. A.3, SPEC's featurizer
# count); QRNN hidden width 64 per direction (the paper does not state it; reading R30).
COND_FEATURES = 227
COND_HIDDEN = 64


def conditioner_numel(in_channels: int, hidden: int, n_layers: int, residual: int) -> int:
    """Length of the conditioner blob in include/dvw.h's order (dvwc_load_weights)."""
    n = 0
    for cin in (in_channels, 2 * hidden):
        n += 2 * (3 * 2 * hidden * cin + 3 * hidden)
    return n + n_layers * 2 * residual * 2 * hidden + n_layers * 2 * residual


def make_conditioner_weights(in_channels: int, hidden: int, n_layers: int, residual: int,
                             seed: int = 0) -> np.ndarray:
    """uniform(+-1/sqrt(fan_in)) per tensor in blob order: fan_in = 2 C_in for the QRNN taps and
    biases (2x1 convolution), 2 hidden for the projections."""
    rng = np.random.default_rng([3, seed])
    parts = []
    for cin in (in_channels, 2 * hidden):
        b = 1.0 / math.sqrt(2 * cin)
        for _ in range(2):  # forward, backward
            parts.append(rng.uniform(-b, b, 3 * 2 * hidden * cin))
            parts.append(rng.uniform(-b, b, 3 * hidden))
    b = 1.0 / math.sqrt(2 * hidden)
    parts.append(rng.uniform(-b, b, n_layers * 2 * residual * 2 * hidden))
    parts.append(rng.uniform(-b, b, n_layers * 2 * residual))
    out = np.concatenate(parts).astype(np.float32)
    assert out.size == conditioner_numel(in_channels, hidden, n_layers, residual)
    return out


def make_features(n_frames: int, in_channels: int = COND_FEATURES, utt: int = 0) -> np.ndarray:
    """Frame-rate features of utterance u: ``default_rng([4, u])``; a one-hot-like phoneme block
    (5 x 45 channels, one active per phoneme slot, held for a random 8-40 frame duration) plus
    a voiced flag and a normalised log-F0 in [-1, 1], padded/truncated to in_channels."""
    rng = np.random.default_rng([4, utt])
    f = np.zeros((n_frames, in_channels), np.float32)
    t = 0
    while t < n_frames:
        d = int(rng.integers(8, 41))
        ph = rng.integers(0, 45, 5)
        voiced = float(rng.random() < 0.7)
        f0 = rng.uniform(-1, 1)
        for k in range(5):
            if 45 * k + ph[k] < in_channels:
                f[t:t + d, 45 * k + ph[k]] = 1.0
        if in_channels > 225:
            f[t:t + d, 225] = voiced
        if in_channels > 226:
            f[t:t + d, 226] = f0 * voiced
        t += d
    return f
