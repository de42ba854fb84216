"""CPU oracle for autoregressive WaveNet sample generation (Deep Voice, arXiv 1702.07825).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
the ``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import,
call, link or execute anything under ``oracle/``.  The product path
(``paper_1702_07825_b200``) never imports this package, and this package never
imports the product's binding or kernels.  The only shared module is
``paper_1702_07825_b200.synth`` (seeded input generators, no method arithmetic),
and this package does not even import that: callers pass the inputs in.

Contents
--------
* ``dvw_oracle.c`` / :func:`run` -- the fp64 ring-buffer oracle (§5.1 steps 1-3,
  App. A.1, App. A.4 direct sampling).  Every step cites PAPER.md in the C file.
* :mod:`oracle.bruteforce` -- a second, independent NumPy fp64 oracle that
  evaluates the dilated causal convolution network over the whole history with
  no ring buffers (the plain definition of App. A.1's ``W * x`` convolutions).
* :mod:`oracle.mulaw` -- mu-law companding closed form (PAPER.md:429 defers to
  WaveNet §2.2; reading R14).
* :mod:`oracle.perfmodel` -- App. E performance model and the parameter roster
  count.

Parity status: the logit *values* for random weights are "parity unpinned by the
paper" (it prints none); they are pinned by agreement of the two independent
oracles, by closed-form special cases and by invariants (tests/test_oracle_*.py).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "dvw_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle (plain C, -O2, no fast-math, no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-ffp-contract=off",
               "-fno-fast-math", "-o", _LIB, _SRC, "-lm"]
        subprocess.check_call(cmd)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        lib.oracle_weights_numel.restype = ctypes.c_int64
        lib.oracle_weights_numel.argtypes = [ctypes.c_int] * 4
        lib.oracle_run.restype = ctypes.c_int
        lib.oracle_run.argtypes = [
            ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
            ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int,
            ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
            ctypes.c_void_p, ctypes.c_void_p,
        ]
        lib.oracle_sample.restype = ctypes.c_int
        lib.oracle_sample.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_float]
        lib.oracle_run_policy.restype = ctypes.c_int
        lib.oracle_run_policy.argtypes = lib.oracle_run.argtypes + [ctypes.c_int, ctypes.c_double, ctypes.c_int]
        lib.oracle_run_nl.restype = ctypes.c_int
        lib.oracle_run_nl.argtypes = lib.oracle_run_policy.argtypes + [ctypes.c_int]
        for fn in ("oracle_appc_tanh", "oracle_appc_sigmoid", "oracle_appc_exp"):
            getattr(lib, fn).restype = ctypes.c_double
            getattr(lib, fn).argtypes = [ctypes.c_double]
        lib.oracle_softmax.restype = None
        lib.oracle_softmax.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
        lib.oracle_sample_policy.restype = ctypes.c_int
        lib.oracle_sample_policy.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                             ctypes.c_int, ctypes.c_float]
        _lib = lib
    return _lib


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def weights_numel(n_layers: int, residual: int, skip: int, levels: int = 256) -> int:
    return int(_load().oracle_weights_numel(n_layers, residual, skip, levels))


def default_dilations(n_layers: int):
    """d_j = 2^((j-1) mod 10) (reading R2)."""
    return [1 << (j % 10) for j in range(n_layers)]


def run(n_layers: int, residual: int, skip: int, weights: np.ndarray, cond: np.ndarray,
        hop: int, n_samples: int, uniforms: Optional[np.ndarray] = None,
        forced: Optional[np.ndarray] = None, levels: int = 256,
        dilations: Optional[Sequence[int]] = None, want_logits: bool = True,
        want_sampled: bool = False, sampler: Optional[tuple] = None, nonlin: str = "exact"):
    """One utterance through the fp64 ring-buffer oracle.

    Returns ``(codes uint8[N], logits float64[N][a] or None, sampled uint8[N] or None)``.
    ``codes[n]`` is the code fed back after step n: ``forced[n]`` when
    teacher-forced, else the inverse-CDF draw with ``uniforms[n]``.  ``sampled[n]``
    is always the draw with ``uniforms[n]`` (for the divergence rate).
    ``sampler = (kind, temperature, top_k)`` selects the App. A.4 strategy (0 direct,
    1 temperature, 2 mean, 3 mode, 4 top-k; see ``sample_policy``); default direct.
    ``nonlin="appc"`` evaluates every tanh, sigma and softmax exp with App. C's
    approximations (``appc_tanh`` / ``appc_sigmoid`` / ``appc_exp``).
    """
    lib = _load()
    w = np.ascontiguousarray(weights, dtype=np.float32)
    c = np.ascontiguousarray(cond, dtype=np.float32)
    assert c.ndim == 3 and c.shape[1] == n_layers and c.shape[2] == 2 * residual, c.shape
    u = None if uniforms is None else np.ascontiguousarray(uniforms, dtype=np.float32)
    f = None if forced is None else np.ascontiguousarray(forced, dtype=np.uint8)
    d = None if dilations is None else np.ascontiguousarray(dilations, dtype=np.int32)
    codes = np.zeros(n_samples, dtype=np.uint8)
    logits = np.zeros((n_samples, levels), dtype=np.float64) if want_logits else None
    sampled = np.zeros(n_samples, dtype=np.uint8) if (want_sampled and u is not None) else None
    kind, temp, topk = sampler if sampler is not None else (0, 1.0, 1)
    nl = {"exact": 0, "appc": 1}[nonlin]
    rc = lib.oracle_run_nl(n_layers, residual, skip, levels, _ptr(d), _ptr(w), w.size, _ptr(c),
                           c.shape[0], hop, _ptr(u), _ptr(f), n_samples, _ptr(codes),
                           _ptr(logits), _ptr(sampled), int(kind), float(temp), int(topk), nl)
    if rc != 0:
        raise ValueError(f"oracle_run rejected its arguments (code {rc})")
    return codes, logits, sampled


def sample(logits: np.ndarray, u: float) -> int:
    """The oracle's inverse-CDF draw on one logit vector (reading R11)."""
    l = np.ascontiguousarray(logits, dtype=np.float64)
    return int(_load().oracle_sample(_ptr(l), l.size, float(np.float32(u))))


def softmax(logits: np.ndarray) -> np.ndarray:
    """p = softmax(l) as the oracle's sampler forms it: e_k = exp(l_k - max l), p_k = e_k / S
    (PAPER.md:374)."""
    l = np.ascontiguousarray(logits, dtype=np.float64)
    p = np.zeros(l.size, dtype=np.float64)
    _load().oracle_softmax(_ptr(l), l.size, _ptr(p))
    return p


DIRECT, TEMPERATURE, MEAN, MODE, TOP_K = 0, 1, 2, 3, 4


def sample_policy(logits: np.ndarray, u: float, kind: int, temperature: float = 1.0, top_k: int = 1) -> int:
    """The oracle's draw under App. A.4 strategy ``kind`` (readings R24-R27):
    temperature P^(1/t)/Z, mean round(E_P[y]), mode argmax (lowest index), top-k (k largest,
    ties by lower index, renormalised); -1 for invalid parameters."""
    l = np.ascontiguousarray(logits, dtype=np.float64)
    return int(_load().oracle_sample_policy(_ptr(l), l.size, int(kind), float(temperature), int(top_k),
                                            float(np.float32(u))))


def appc_tanh(x: float) -> float:
    """App. C tanh: sign(x) (e~ - 1/e~) / (e~ + 1/e~), e~ = 1 + |x| + 0.5658 x^2 + 0.143 x^4
    (PAPER.md:556, 567)."""
    return float(_load().oracle_appc_tanh(float(x)))


def appc_sigmoid(x: float) -> float:
    """App. C sigma: e~ / (1 + e~) for x >= 0, 1 / (1 + e~) for x <= 0."""
    return float(_load().oracle_appc_sigmoid(float(x)))


def appc_exp(x: float) -> float:
    """App. C.2 e^x (x <= 0): the fp32 bit pattern I = (x/ln2 + 126 + g(z)) 2^23 with the
    rational g (reading R31)."""
    return float(_load().oracle_appc_exp(float(x)))
