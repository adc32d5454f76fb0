"""Calibrated analytic model: the reference's decode_ttl
(latency.cpp:207-250, restated in paper_2507_07120_b200/analytic.py and pinned
to the reference's own library by tests/test_analytic.py) evaluated with a
HardwareSpec MEASURED on this B200, next to the measured decode step.

    python tools/calibrate.py BENCH_JSON [--out profiles/r02_calibration.md]

Measured HardwareSpec ("b200-calibrated"):
  * mem_bw             = the attention kernel's achieved HBM bandwidth (the
                         bench line's roofline.achieved) -- what a streaming
                         kernel of this engine actually sustains;
  * compute_throughput = the MLA kernel's achieved tensor throughput
                         (deepseek_slice.mla_attention), else the sustained
                         cuBLAS bf16 figure of MEASURED_PEAKS.json;
  * link_bw / latency  = NVLink 5 nominal (900 GB/s, 0.1 us): one GPU here;
  * bytes_per_param    = 2 (bf16 weights and KV, as measured).
Each configuration the bench line measured is then simulated per component
(QKV, KV read, O-projection, FFN) and whole step, and the ratio
measured / simulated says where the B200 step departs from the model.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2507_07120_b200 import analytic as A  # noqa: E402
from paper_2507_07120_b200.model import PRESETS, HardwareSpec, ParallelismConfig  # noqa: E402


def measured_hw(line):
    att = line["roofline"]
    bw = att["achieved"] * 1e9
    tc = None
    mla = line.get("deepseek_slice", {}).get("mla_attention", {}).get("roofline")
    if mla:
        tc = mla["achieved"] * 1e12
    if tc is None:
        try:
            with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
                tc = json.load(f)["bf16_tflops_sustained"] * 1e12
        except Exception:
            tc = 1.393e15
    return HardwareSpec("b200-calibrated", bw, tc, 9e11, 1e-7, 64, 2.0, 180e9)


def with_layers(spec, layers):
    from dataclasses import replace
    return replace(spec, layers=layers)


def rows_for(line, hw):
    out = []
    # configs[1]: llama3-8b-like, one GPU, B = 8, S = 131072, 32 layers (+ LM head, outside the model)
    spec = PRESETS["llama3-8b-like"]
    cfg = ParallelismConfig("helix", 1, 1, 1, 1, 1)
    B, S, L = line["config"]["global_batch"], line["config"]["seq_len"], line["config"]["layers"]
    b = A.decode_ttl(cfg, with_layers(spec, L), B, S, hw, hopb=True)
    br = line["breakdown_ms"]
    out.append({"config": f"C2 llama3-8b-like 1 GPU B={B} S={S} ({L} layers)",
                "components_ms": {
                    "qkv": (b.qkv_proj * L * 1e3, br["qkv"]),
                    "attention (kv read)": (max(b.kv_read, b.attn_compute) * L * 1e3,
                                            br["attention"] + br["split_reduce"] + br.get("merge", 0.0)),
                    "o_proj": (b.post_proj * L * 1e3, br["o_proj"]),
                    "ffn": (max(b.ffn_weight_read, b.ffn_compute) * L * 1e3, br["gate_up"] + br["down"]),
                },
                "step_ms": (b.ttl * 1e3, line["ms_per_step"] - br["lm_head"] - br["embed"])})
    # configs[1] at KVP = 2/4/8 (one GPU of the pool, collectives modeled)
    for n, k in sorted(line.get("kvp_slices", {}).items()):
        if not isinstance(k, dict) or "ttl_ms_compute" not in k:
            continue
        n = int(n)
        cfgn = ParallelismConfig("helix", 1, n, n, 1, 1)
        bn = A.decode_ttl(cfgn, with_layers(spec, L), B, k["global_context"], hw, hopb=True)
        out.append({"config": f"C2 model at KVP={n} (one GPU of the pool, S_global={k['global_context']})",
                    "step_ms": (bn.ttl * 1e3, k["ttl_ms_compute"])})
    # configs[2] / [3]: one layer of one GPU of the KVP = 8 pool
    for key, preset, cfgn in (("llama405b_slice", "llama405b-like", ParallelismConfig("helix", 1, 8, 8, 1, 1)),
                              ("deepseek_slice", "deepseek-r1-like", ParallelismConfig("helix", 1, 8, 1, 8, 1))):
        sl = line.get(key)
        if not isinstance(sl, dict) or "ms_per_layer" not in sl:
            continue
        s_glob = sl["kv_tokens_per_request_on_this_gpu"] * 8
        bl = A.decode_ttl(cfgn, with_layers(PRESETS[preset], 1), B, s_glob, hw, hopb=True)
        m = sl["breakdown_ms"]
        out.append({"config": f"{key}: {preset} layer, one GPU of KVP=8, S_global={s_glob}",
                    "components_ms": {
                        "qkv": (bl.qkv_proj * 1e3, m["qkv"]),
                        "attention": (max(bl.kv_read, bl.attn_compute) * 1e3, m["attention"] + m["split_reduce"]),
                        "o_proj": (bl.post_proj * 1e3, m["o_proj"]),
                        "ffn": (max(bl.ffn_weight_read, bl.ffn_compute) * 1e3,
                                m["gate_up_or_router_to_gate_up"] + m["down_or_down_combine"]),
                    },
                    "layer_ms": ((bl.ttl - A.comm_time("broadcast", 8, B * 16384 * 2, hw)) * 1e3,
                                 sl["ms_per_layer"] - m["lm_head"] - m["embed"])})
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("bench_json")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    with open(a.bench_json) as f:
        line = json.loads(f.read().strip().splitlines()[-1])
    hw = measured_hw(line)
    rows = rows_for(line, hw)
    md = ["# Calibrated analytic model vs measured (tools/calibrate.py)", "",
          f"Source: `{os.path.relpath(a.bench_json, ROOT)}`. Measured HardwareSpec: mem_bw "
          f"{hw.mem_bw / 1e9:.0f} GB/s (attention kernel achieved), compute {hw.compute_throughput / 1e12:.0f} TF/s "
          "(MLA kernel achieved), NVLink nominal 900 GB/s / 0.1 us, 2 B/param. The model is the reference's "
          "decode_ttl (latency.cpp:207-250) restated in analytic.py, pinned to the reference library.", "",
          "| configuration | component | simulated ms | measured ms | measured / simulated |", "|---|---|---|---|---|"]
    for r in rows:
        for comp, (sim, meas) in r.get("components_ms", {}).items():
            md.append(f"| {r['config']} | {comp} | {sim:.3f} | {meas:.3f} | {meas / sim:.2f} |")
        for k in ("step_ms", "layer_ms"):
            if k in r:
                sim, meas = r[k]
                md.append(f"| {r['config']} | **{k.replace('_ms', '')}** | {sim:.3f} | {meas:.3f} | "
                          f"{meas / sim:.2f} |")
    text = "\n".join(md) + "\n"
    print(text)
    if a.out:
        with open(a.out, "w") as f:
            f.write(text)
        with open(os.path.splitext(a.out)[0] + ".json", "w") as f:
            json.dump({"hardware": hw.to_json(), "rows": rows}, f, indent=1)


if __name__ == "__main__":
    main()
