"""Summarise an ncu --page source --csv (SASS) export: stall samples by region
and reason, top stalled instructions.  python tools/ncu_stalls.py src.csv [bin]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
iS = h.index('Source')
iN = h.index('Warp Stall Sampling (All Samples)')
iE = h.index('Instructions Executed')
reasons = [c for c in h if c.startswith('stall_') and 'Not Issued' not in c]
ri = [h.index(c) for c in reasons]
data = []
for r in rows[2:]:
    try:
        n = float(r[iN] or 0)
        e = float(r[iE] or 0)
    except (ValueError, IndexError):
        continue
    data.append((n, r[iS], e, [float(r[i] or 0) for i in ri]))
tot = sum(d[0] for d in data)
B = int(sys.argv[2]) if len(sys.argv) > 2 else 120
print('total samples', tot)
for b in range(0, len(data), B):
    seg = data[b:b + B]
    ns = sum(x[0] for x in seg)
    if ns / tot < 0.01:
        continue
    rs = [sum(x[3][k] for x in seg) for k in range(len(reasons))]
    top = sorted(zip(rs, reasons), reverse=True)[:4]
    ops = sorted(set(x[1].split()[0] if not x[1].startswith('@') else x[1].split()[1] for x in seg
                     if any(t in x[1] for t in ['F2FP', 'UTC', 'LDTM', 'STTM', 'MUFU', 'LDS', 'STS', 'SYNCS', 'BAR', 'UBLKCP', 'HMUL2', 'PRMT', 'SHFL'])))
    print(f"{b:5d} {100 * ns / tot:5.1f}%  " + ", ".join(f"{n[6:]} {100 * v / tot:.1f}" for v, n in top) + "  | " + " ".join(ops[:9]))
