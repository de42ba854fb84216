"""App. E performance model and parameter roster (TEST INFRASTRUCTURE ONLY).

PAPER.md:608-630 (App. E):
  Cost(layer)  = 10 r^2 + 11 r + 2 r (f_d + f_e)
  Cost(sample) = l (10 r^2 + 11 r + 2 r (f_d + f_e)) + s (2 r l + 2)
                 + a (2 s + 2 a + 3) + a (3 + f_d + f_e)
  with l = 40, r = 64, s = a = 256, f_d = f_e = 10 and 16,384 Hz: ~55e9 FLOP/s.
PAPER.md:227 (§5): "approximately 1.6e6 parameters ... about 6.4 MB".
"""
from __future__ import annotations


def cost_layer(r: int, f_d: int = 10, f_e: int = 10) -> int:
    return 10 * r * r + 11 * r + 2 * r * (f_d + f_e)


def cost_sample(L: int, r: int, s: int, a: int = 256, f_d: int = 10, f_e: int = 10) -> int:
    return (L * cost_layer(r, f_d, f_e) + s * (2 * r * L + 2) + a * (2 * s + 2 * a + 3)
            + a * (3 + f_d + f_e))


def n_params(L: int, r: int, s: int, a: int = 256) -> int:
    """Per layer W_prev, W_cur (2r x r), B (2r), W_res (r x r), B_res (r), W_skip (s x r);
    global W_emb_prev, W_emb_cur (r x a), B_emb (r), B_skip (s), W_relu (a x s),
    B_relu (a), W_out (a x a), B_out (a)."""
    per_layer = 2 * (2 * r * r) + 2 * r + r * r + r + s * r
    return L * per_layer + 2 * r * a + r + s + a * s + a + a * a + a


def macs_per_sample(L: int, r: int, s: int, a: int = 256) -> int:
    """Multiply-accumulates of the matvecs alone: l(5r^2 + r s) + a s + a^2."""
    return L * (5 * r * r + r * s) + a * s + a * a


def receptive_field(dilations) -> int:
    """R = 2 + sum_j d_j: the embedding's 2x1 conv reaches two codes back, each
    dilated layer adds d_j (SPEC receptive_field)."""
    return 2 + int(sum(dilations))
