"""Oracle of the int16 / int8 weight tier (row f4; "inference with weight
matrices quantized to int16"; reading R32).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): only tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs may use it.  It shares no code with the CUDA
path: the roster below is restated from the blob layout (dvw_oracle.c header), not imported.

The paper gives no scheme.  Reading R32: every weight MATRIX is quantised symmetrically per
row (biases stay fp32):
    s = max_c |W[row][c]| / (2^(bits-1) - 1)      (fp32 division)
    q = rint(W[row][c] / s)                        (fp32 division, round half to even)
    W[row][c] := q * s                              (fp32 product)
A row of zeros stays zero.

Reading R33 (the per-tensor alternative, SPEC.md's QuantizedWeightSet): one scale per weight
matrix, s = max |W| / (2^(bits-1) - 1), s = 1 for an all-zero matrix, q = rint(W / s),
W := q s, same fp32 arithmetic.  The integer code q is a decision floating point takes, so it is
taken in the kernel's precision (fp32) -- here with numpy float32 scalars and arrays, whose
division and product are the IEEE single-precision operations.
"""
import numpy as np


def roster(L: int, r: int, s: int, a: int = 256):
    """(offset, rows, cols) of every weight matrix in the blob, in blob order."""
    mats = []
    p = 0
    for _ in range(L):
        mats.append((p, 2 * r, r)); p += 2 * r * r      # W_prev
        mats.append((p, 2 * r, r)); p += 2 * r * r      # W_cur
        p += 2 * r                                      # B
        mats.append((p, r, r)); p += r * r              # W_res
        p += r                                          # B_res
        mats.append((p, s, r)); p += s * r              # W_skip
    mats.append((p, r, a)); p += r * a                  # W_emb_prev
    mats.append((p, r, a)); p += r * a                  # W_emb_cur
    p += r + s                                          # B_emb, B_skip
    mats.append((p, a, s)); p += a * s                  # W_relu
    p += a                                              # B_relu
    mats.append((p, a, a)); p += a * a                  # W_out
    p += a                                              # B_out
    return mats, p


def quantize_rows(W: np.ndarray, bits: int) -> np.ndarray:
    """Per-row symmetric quantise-dequantise of a float32 matrix (reading R32)."""
    W = np.asarray(W, dtype=np.float32)
    qmax = np.float32((1 << (bits - 1)) - 1)
    out = W.copy()
    for i in range(W.shape[0]):
        m = np.float32(np.max(np.abs(W[i])))
        if m == 0:
            continue
        sc = np.float32(m / qmax)
        out[i] = (np.rint(W[i] / sc) * sc).astype(np.float32)
    return out


def quantize_codes(W: np.ndarray, bits: int):
    """The integer codes and scales behind quantize_rows (for the pins)."""
    W = np.asarray(W, dtype=np.float32)
    qmax = np.float32((1 << (bits - 1)) - 1)
    m = np.max(np.abs(W), axis=1).astype(np.float32)
    sc = np.where(m > 0, m / qmax, np.float32(1)).astype(np.float32)
    return np.rint(W / sc[:, None]).astype(np.int64), sc


def quantize_tensor_codes(W: np.ndarray, bits: int):
    """Per-tensor symmetric codes and scale (reading R33): (q int64, s float32)."""
    W = np.asarray(W, dtype=np.float32)
    qmax = np.float32((1 << (bits - 1)) - 1)
    m = np.float32(np.max(np.abs(W))) if W.size else np.float32(0)
    sc = np.float32(m / qmax) if m > 0 else np.float32(1)
    return np.rint(W / sc).astype(np.int64), sc


def quantize_tensor(W: np.ndarray, bits: int) -> np.ndarray:
    """Per-tensor symmetric quantise-dequantise (reading R33)."""
    q, sc = quantize_tensor_codes(W, bits)
    return (q.astype(np.float32) * sc).astype(np.float32)


def quantize_weights(blob: np.ndarray, L: int, r: int, s: int, bits: int, a: int = 256,
                     scheme: str = "per_row") -> np.ndarray:
    """The whole blob with every weight matrix quantised; biases unchanged.
    scheme: "per_row" (R32) or "per_tensor" (R33)."""
    fn = {"per_row": quantize_rows, "per_tensor": quantize_tensor}[scheme]
    w = np.array(blob, dtype=np.float32, copy=True)
    mats, numel = roster(L, r, s, a)
    assert w.size == numel, (w.size, numel)
    for off, rows, cols in mats:
        w[off:off + rows * cols] = fn(w[off:off + rows * cols].reshape(rows, cols), bits).ravel()
    return w
