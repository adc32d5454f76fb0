"""CPU: the oracle's FP4 (e2m1) KV block rounding (helix_oracle.cpp
round_e2m1_block), pinned against an independent brute-force restatement of
the OCP MX e2m1 element format (grid {0, 0.5, 1, 1.5, 2, 3, 4, 6}, round to
nearest, ties to the even code, saturating) with a shared power-of-two block
scale -- the storage the B200 kernels decode (fp8.cuh e2m1_*). The reference
evaluates Helix at FP4 but has no FP4 numerics of its own."""
import math

import numpy as np

from tests import oracle_py as O

GRID = np.array([0.0, 0.5, 1.0, 1.5, 2.0, 3.0, 4.0, 6.0])


def independent(block):
    amax = float(np.abs(block).max())
    if amax > 0:
        e = math.ceil(math.log2(amax / 6.0))
        # exact power-of-two boundary: log2 may round; fix up to the smallest e with 6 * 2^e >= amax
        while 6.0 * 2.0 ** (e - 1) >= amax:
            e -= 1
        while 6.0 * 2.0 ** e < amax:
            e += 1
        e = min(13, max(-14, e))
    else:
        e = 0
    out = np.empty_like(block)
    for i, x in enumerate(block):
        t = abs(x) / 2.0 ** e
        d = np.abs(GRID - t)
        cand = np.flatnonzero(d == d.min())
        code = cand[0] if len(cand) == 1 else [c for c in cand if c % 2 == 0][0]
        out[i] = math.copysign(GRID[code] * 2.0 ** e, x)
    return out


def test_e2m1_block_rounding_matches_independent_restatement():
    rng = np.random.default_rng(0)
    blocks = [rng.uniform(-1, 1, 32), rng.normal(0, 3, 32), rng.uniform(-1e-4, 1e-4, 32), np.zeros(32),
              rng.uniform(-100, 100, 32) * (rng.uniform(size=32) < 0.1)]
    # exact grid points, midpoints (ties), the saturation edge and the block max on a power of two
    t = np.array([0.25, 0.75, 1.25, 1.75, 2.5, 3.5, 5.0, 6.0, 0.5, 1.0, 3.0, 4.0] * 2 + [6.0] * 8)
    for e in (-3, 0, 2):
        blocks.append(t * 2.0 ** e * np.where(np.arange(32) % 3 == 0, -1.0, 1.0))
    for _ in range(200):
        blocks.append(rng.uniform(-1, 1, 32) * 2.0 ** rng.integers(-12, 8))
    for b in blocks:
        np.testing.assert_array_equal(O.round_e2m1_block(b), independent(b))


def test_e2m1_values_are_exact_in_f16():
    """Every stored value grid * 2^e (e in [-14, 13]) is representable in f16 --
    the kernels widen codes with cvt.rn.f16x2.e2m1x2 and multiply by 2^e in f16."""
    for e in range(-14, 14):
        v = GRID * 2.0 ** e
        np.testing.assert_array_equal(v.astype(np.float16).astype(np.float64), v)


def test_fp4_weights_oracle_quantisation():
    """ModelDims::w_fp4 (layer_oracle.cpp quantize_fp4_cols): every GEMV weight
    column (output feature) n is stored in e2m1 blocks of 32 consecutive inputs
    k = 32 i .. 32 i + 31 with a power-of-two block scale -- the same MX rounding
    as the KV pages, checked here against the independent restatement over the
    unquantised draws of the bf16=False oracle."""
    H, Q, K, D, F, V = 64, 4, 2, 16, 96, 50
    q4 = O.Model(H, Q, K, D, F, 1, V, seed=9, qkv_hash=True, w_fp4=True)
    ref = O.Model(H, Q, K, D, F, 1, V, seed=9, qkv_hash=True, bf16=False)
    for name in ("wq", "wk", "wv", "wo", "wgate", "wup", "wdown", "lm"):
        w, w0 = q4.weight(name), ref.weight(name)
        assert w.shape == w0.shape and w.shape[0] % 32 == 0
        want = np.empty_like(w0)
        for n in range(w0.shape[1]):
            for k0 in range(0, w0.shape[0], 32):
                want[k0:k0 + 32, n] = independent(w0[k0:k0 + 32, n])
        np.testing.assert_array_equal(w, want)
