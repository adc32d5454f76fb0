"""Run the bench's deepseek-r1-like single-GPU slice once (for ncu captures)."""
import sys
sys.path.insert(0, ".")
import bench  # noqa: E402


class A:
    batch, deepseek_context, warmup, steps = 8, 125000, 2, 2


print(bench.deepseek_slice(A())["breakdown_ms"])
