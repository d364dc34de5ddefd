"""Aggregate an `ncu --page source --csv --print-source cuda,sass` export by CUDA source line:
warp-stall samples per line plus the dominant stall reasons (for reading profiles here)."""
import csv
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
rows = list(csv.reader(open(path)))
cur_file = None
agg = {}
hdr = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] in ("", "Function Name"):
        continue
    try:
        samp = float(r[4])
    except ValueError:
        continue
    stalls = {}
    for i, name in enumerate(hdr):
        if name.startswith("stall_") and i < len(r):
            try:
                stalls[name[6:]] = float(r[i])
            except ValueError:
                pass
    key = (cur_file, int(r[0]))
    a = agg.setdefault(key, [0.0, r[1].strip()[:100], {}])
    a[0] += samp
    for k, v in stalls.items():
        a[2][k] = a[2].get(k, 0.0) + v
tot = sum(v[0] for v in agg.values()) or 1.0
print(f"total samples {tot:.0f}")
for (f, ln), (v, src, st) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    reasons = ", ".join(f"{k} {100*x/v:.0f}%" for k, x in sorted(st.items(), key=lambda kv: -kv[1])[:3] if v and x > 0)
    print(f"{100*v/tot:5.1f}% {f}:{ln}: {src}  [{reasons}]")
