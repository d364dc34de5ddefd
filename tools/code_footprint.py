"""Executed-code footprint per source line from an ncu source export
(`ncu -i R --page source --csv --print-source cuda,sass > f.csv`): how many distinct SASS
instructions each line executed (instruction-cache footprint) and its stall samples."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
fp = collections.Counter(); smp = collections.Counter(); ffp = collections.Counter(); src = {}
addrs = set()
f = line = None
for r in rows:
    if r and r[0] == "File Path": f = r[1].split("/")[-1]; continue
    if not r or r[0] in ("Function Name", "Line No"): continue
    if r[0]:
        if not r[0].isdigit() or len(r) < 8: continue
        line = (f, int(r[0])); src[line] = r[1].strip()[:70]; smp[line] += int(r[4]) if r[4].isdigit() else 0
        continue
    if len(r) > 7 and r[2].startswith("0x") and r[7].isdigit() and int(r[7]) > 0:
        a = int(r[2], 16)
        if a not in addrs:
            addrs.add(a); fp[line] += 1; ffp[line[0]] += 1
print("executed static SASS:", len(addrs), "instructions,", len(addrs) * 16 // 1024, "KB;",
      "128B lines:", len({a // 128 for a in addrs}))
print("per file:", dict(ffp))
for (fl, ln), n in fp.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 40):
    print(f"{n:5d} {smp[(fl, ln)]:4d}  {fl}:{ln}  {src[(fl, ln)]}")
