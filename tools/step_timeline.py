"""Kernel timeline of decode steps (CUPTI via torch.profiler / kineto): start,
end and duration of every kernel of two graph-replayed steps of configs[1]'s
model (llama3-8b-like, B = 8, 32 layers), PDL overlap included -- unlike an ncu
launch list, which serialises the kernels. Prints the first ~60 kernels and the
per-kernel totals; --layer-path prints the per-layer critical path (how long
after its predecessor's end each kernel ends).

    python tools/step_timeline.py [--context 131072] [--w bf16] [--kv bf16] [--layer-path]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--context", type=int, default=131072)
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--w", default="bf16")
    ap.add_argument("--kv", default="bf16")
    ap.add_argument("--rows", type=int, default=60)
    ap.add_argument("--layer-path", action="store_true")
    a = ap.parse_args()
    import torch
    from torch.profiler import profile, ProfilerActivity
    import paper_2507_07120_b200 as P
    spec = P.model.PRESETS["llama3-8b-like"]
    B = 8
    g = P.HelixDecoder(spec, batch=B, capacity=a.context + 256, layers=a.layers, w_dtype=a.w, kv_dtype=a.kv)
    g.init_weights(2507, qkv="hash")
    g.fill_kv_hash(a.context, 2507)
    tok = torch.randint(0, spec.vocab, (B,), dtype=torch.int32, device="cuda")
    nxt = torch.zeros(B, dtype=torch.int32, device="cuda")
    for _ in range(5):
        g.step_device(tok.data_ptr(), nxt.data_ptr())
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(2):
            g.step_device(tok.data_ptr(), nxt.data_ptr())
        torch.cuda.synchronize()
    evs = sorted((e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA),
                 key=lambda e: e.time_range.start)
    t0 = evs[0].time_range.start
    rows = [(e.time_range.start - t0, e.time_range.end - t0, e.name.replace("hx::", "")[:64]) for e in evs]
    print(f"# {len(rows)} kernels over {rows[-1][1] - rows[0][0]:.1f} us (2 steps), context {a.context}, "
          f"w {a.w}, kv {a.kv}")
    print("| start (us) | end (us) | dur (us) | end - previous end (us) | kernel |\n|---|---|---|---|---|")
    prev_end = 0.0
    for s0, s1, n in rows[:a.rows]:
        print(f"| {s0:.1f} | {s1:.1f} | {s1 - s0:.1f} | {s1 - prev_end:+.1f} | `{n}` |")
        prev_end = max(prev_end, s1)
    agg = {}
    for s0, s1, n in rows:
        x = agg.setdefault(n, [0.0, 0])
        x[0] += s1 - s0
        x[1] += 1
    print("\n| total dur (us) | launches | kernel |\n|---|---|---|")
    for n, (d, c) in sorted(agg.items(), key=lambda x: -x[1][0]):
        print(f"| {d:.1f} | {c} | `{n}` |")


if __name__ == "__main__":
    main()
