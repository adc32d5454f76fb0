"""Summarise ncu outputs into profiles/ (tracked). Usage:
    python profiles/summarize.py launches <launches.csv> <out.md>
    python profiles/summarize.py full <report.ncu-rep> <out.md> [<summary.json>]
    python profiles/summarize.py hopb <hopb_sweep.jsonl> <out.md>
"""
import csv
import io
import json
import subprocess
import sys

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
           "launch__grid_size", "launch__waves_per_multiprocessor", "launch__occupancy_limit_shared_mem"]


def launches(path, out):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    ix = {h: i for i, h in enumerate(rows[hi])}
    agg = {}
    for r in rows[hi + 1:]:
        key = (int(r[ix["ID"]]), r[ix["Kernel Name"]])
        agg.setdefault(key, {})[r[ix["Metric Name"]]] = float(r[ix["Metric Value"]].replace(",", ""))
    lines = ["| id | kernel | time (us) | DRAM read (MB) | GB/s |", "|---|---|---|---|---|"]
    total = 0.0
    for (i, n), m in sorted(agg.items()):
        t = m.get("gpu__time_duration.sum", 0.0)
        b = m.get("dram__bytes_read.sum", 0.0)
        total += t
        lines.append(f"| {i} | `{n[:60]}` | {t / 1e3:.1f} | {b / 1e6:.1f} | {b / max(t, 1):.0f} |")
    lines.append(f"\nsum of kernel durations: {total / 1e6:.3f} ms (serialised, cold-cache: compare shares)")
    open(out, "w").write("\n".join(lines) + "\n")


def full(rep, out, summary=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = rows[0]
    lines = []
    js = {}
    for row in rows[2:]:
        name = row[hdr.index("Kernel Name")]
        lines.append(f"### `{name}`")
        d = {}
        for m in METRICS:
            if m in hdr:
                lines.append(f"- {m} = {row[hdr.index(m)]}")
                try:
                    d[m] = float(row[hdr.index(m)].replace(",", ""))
                except ValueError:
                    pass
        js.setdefault(name, d)
    open(out, "w").write("\n".join(lines) + "\n")
    if summary:
        att = next((v for k, v in js.items() if "attn_decode" in k), None)
        if att:
            # ncu reports dram bytes in the unit of the raw page (Gbyte / Mbyte rows); normalise via time x throughput
            json.dump({"attention": {"dram_bytes_per_launch": att.get("dram_bytes_read_total")}}, open(summary, "w"))


def hopb(path, out):
    rows = [json.loads(l) for l in open(path) if l.strip()]
    ok = [r for r in rows if "attn_ms_off" in r]
    for r in ok:  # both modes end with the same flag wait (older records counted it on one side only)
        if abs(r["exposed_a2a_ms_off"] - r["a2a_ms_modeled"]) < 1e-12:
            r["exposed_a2a_ms_off"] += r["flag_wait_ms_off"]
            r["hopb_gain_ms"] = (r["attn_ms_off"] + r["exposed_a2a_ms_off"]) - (r["attn_ms_on"] + r["exposed_a2a_ms_on"])
    on_hdr = "attn + stream reducer on (ms, serialised)" if any("attn_kernel_ms_on" in r for r in ok) \
        else "attn, in-kernel push on (ms)"
    lines = [f"| KVP | context | B | KV tok/GPU | attn+reduce off (ms) | {on_hdr} | layer off (ms) | "
             "layer on (ms) | a2a modeled (us) | exposed off (us) | exposed on (us) | hidden | HOP-B net (us) |",
             "|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
    for r in ok:
        hf = r.get("a2a_hidden_frac")
        lines.append(f"| {r['kvp']} | {r['context']} | {r['batch']} | {r['kv_tokens_per_gpu']} | "
                     f"{r['attn_ms_off']:.3f} | {r['attn_ms_on']:.3f} | {r['layer_ms_off']:.3f} | "
                     f"{r['layer_ms_on']:.3f} | {r['a2a_ms_modeled'] * 1e3:.2f} | {r['exposed_a2a_ms_off'] * 1e3:.2f} | "
                     f"{r['exposed_a2a_ms_on'] * 1e3:.2f} | {'-' if hf is None else f'{hf:.2f}'} | "
                     f"{r['hopb_gain_ms'] * 1e3:+.1f} |")
    for r in rows:
        if "skipped" in r or "error" in r:
            lines.append(f"| {r['kvp']} | {r['context']} | {r['batch']} | {r.get('skipped') or r.get('error')} |"
                         " | | | | | | | | |")
    open(out, "w").write("\n".join(lines) + "\n")


if __name__ == "__main__":
    if sys.argv[1] == "hopb":
        hopb(sys.argv[2], sys.argv[3])
    elif sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        full(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else None)
