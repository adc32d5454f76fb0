"""Run one of the bench's one-GPU-of-8 slices once (for ncu captures).

    python tools/ds_slice.py [deepseek-r1-like|llama405b-like] [w_dtype] [kv_dtype]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


class A:
    batch, warmup, steps = 8, 2, 2


preset = sys.argv[1] if len(sys.argv) > 1 else "deepseek-r1-like"
w_dtype = sys.argv[2] if len(sys.argv) > 2 else "bf16"
kv_dtype = sys.argv[3] if len(sys.argv) > 3 else "bf16"
print(bench.pool_slice(A(), preset, 125000, 8 if preset == "deepseek-r1-like" else 1, w_dtype, kv_dtype)["breakdown_ms"])
