"""mu-law companding with a = 256 levels (TEST INFRASTRUCTURE ONLY).

PAPER.md:429 (App. A.1): "Audio is quantized to a=256 values using mu-law
companding, as described in Section 2.2 of WaveNet" -- the paper defers to
WaveNet's closed form F(x) = sign(x) ln(1 + mu|x|) / ln(1 + mu), mu = a - 1.
The rounding rule is unstated; reading R14 takes the torchaudio convention
(pinned against torchaudio.functional in tests/test_oracle_pins.py):
    encode: c = floor((F(x) + 1) / 2 * mu + 0.5)
    decode: g = 2 c / mu - 1 ; x = sign(g) ((1 + mu)^|g| - 1) / mu
"""
from __future__ import annotations

import numpy as np


def encode(x, levels: int = 256) -> np.ndarray:
    mu = levels - 1
    x = np.clip(np.asarray(x, dtype=np.float64), -1.0, 1.0)
    f = np.sign(x) * np.log1p(mu * np.abs(x)) / np.log1p(mu)
    return np.floor((f + 1.0) / 2.0 * mu + 0.5).astype(np.int64)


def decode(c, levels: int = 256) -> np.ndarray:
    mu = levels - 1
    g = 2.0 * np.asarray(c, dtype=np.float64) / mu - 1.0
    return np.sign(g) * (np.power(1.0 + mu, np.abs(g)) - 1.0) / mu
