"""Summarise an ncu source page (--print-source=cuda,sass) by CUDA source line: stall samples and
instructions executed.  Usage: ncu -i rep --page source --csv --print-source=cuda,sass > f.csv;
python tools/ncu_hot.py f.csv [top]"""
import csv, sys, collections
path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
rows = list(csv.reader(open(path)))
cur_file = None
agg = collections.defaultdict(lambda: [0, 0, ""])
hdr = None
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8 or not r[0].isdigit():
        continue
    try:
        line = int(r[0]); stall = int(r[4] or 0); inst = int(r[7] or 0)
    except ValueError:
        continue
    key = (cur_file, line)
    agg[key][0] += stall
    agg[key][1] += inst
    if not agg[key][2]:
        agg[key][2] = r[1][:90]
tot_s = sum(v[0] for v in agg.values()) or 1
tot_i = sum(v[1] for v in agg.values()) or 1
print(f"total stall samples {tot_s}, instructions {tot_i}")
for (f, l), (s, i, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100*s/tot_s:5.1f}% stall {100*i/tot_i:5.1f}% inst  {f}:{l}  {src}")
