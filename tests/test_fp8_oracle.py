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
