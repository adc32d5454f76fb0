"""CPU: the oracle's FP8 E4M3 rounding (helix_oracle.cpp round_e4m3) -- the
checker behind the GPU's optional FP8 KV pages -- against an independent
implementation, torch.float8_e4m3fn (RNE; saturation applied by clamping to
+-448 first, the cvt.rn.satfinite semantics the B200 path uses)."""
import numpy as np
import pytest

from tests import oracle_py as O


def torch_e4m3(x):
    torch = pytest.importorskip("torch")
    t = torch.tensor(x, dtype=torch.float32).clamp(-448.0, 448.0)
    return t.to(torch.float8_e4m3fn).to(torch.float64).numpy()


def test_round_e4m3_matches_torch():
    rng = np.random.default_rng(0)
    xs = np.concatenate([
        np.linspace(-500, 500, 20001), np.linspace(-1, 1, 20001),
        rng.standard_normal(50000) * np.logspace(-4, 3, 50000),
        # binade edges, subnormals, ties and saturation
        np.array([2.0 ** -10, 2.0 ** -9 * 1.5, 2.0 ** -9 * 2.5, 2.0 ** -6 * (1 - 1 / 32), 448.0, 449.0,
                  463.99, 464.0, 480.0, 1e6, -1e-12, 0.0, 1.0625, 1.1875, -3.75])])
    xs = xs.astype(np.float32).astype(np.float64)  # exactly representable for the torch path
    np.testing.assert_array_equal(O.round_e4m3(xs), torch_e4m3(xs))


def test_round_e4m3_grid():
    # every finite e4m3 value is a fixed point; the largest is 448, the smallest subnormal 2^-9
    vals = [m * 2.0 ** -9 for m in range(8)] + [(1 + m / 8) * 2.0 ** e for e in range(-6, 9) for m in range(8)]
    vals = [v for v in vals if v <= 448.0]
    np.testing.assert_array_equal(O.round_e4m3(vals), np.array(vals))
    assert O.round_e4m3([1e30])[0] == 448.0 and O.round_e4m3([-1e30])[0] == -448.0


def test_fp8_weights_oracle_quantisation():
    """ModelDims::w_fp8 (layer_oracle.cpp hash_matrix_fp8): each GEMV weight column
    (output feature) n is e4m3(W / s_n) * s_n with s_n the smallest power of two
    >= max_k |W[k][n]| / 448; the unquantised draws come from the bf16=False oracle."""
    H, Q, K, D, F, V = 64, 4, 2, 16, 96, 50
    q8 = O.Model(H, Q, K, D, F, 1, V, seed=9, qkv_hash=True, w_fp8=True)
    ref = O.Model(H, Q, K, D, F, 1, V, seed=9, qkv_hash=True, bf16=False)
    for name in ("wq", "wk", "wv", "wo", "wgate", "wup", "wdown", "lm"):
        w, w0 = q8.weight(name), ref.weight(name)
        amax = np.abs(w0).max(axis=0)
        s = np.exp2(np.ceil(np.log2(amax / 448.0)))
        np.testing.assert_array_equal(w, O.round_e4m3(w0 / s) * s)
        assert np.all(np.abs(w / s).max(axis=0) <= 448.0)
        assert np.all(np.abs(w / s).max(axis=0) > 224.0 * 0.9)  # the scale is the smallest power of two


def test_mla_query_quantisation_matches_torch():
    """The FP8-latent MLA query image (layer_oracle.cpp quantize_q_e4m3_pow2, the
    rule of the GPU's absorb kernel, mla.cu Q8): per head, e = the largest exponent
    with max |q| * 2^e <= 448, values e4m3(q * 2^e) * 2^-e -- against torch.float8_e4m3fn."""
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(3)
    for scale in (1e-6, 3e-3, 0.7, 1.0, 5.0, 448.0, 1e3, 2.0 ** 20):
        q = (rng.standard_normal(576) * scale).astype(np.float32).astype(np.float64)
        got, e = O.quantize_q_e4m3_pow2(q)
        mx = np.abs(q).max()
        assert mx * 2.0 ** e <= 448.0 < mx * 2.0 ** (e + 1)
        want = torch_e4m3(q * 2.0 ** e) * 2.0 ** -e
        np.testing.assert_array_equal(got, want)
    got, e = O.quantize_q_e4m3_pow2(np.zeros(576))
    assert e == 0 and not got.any()
