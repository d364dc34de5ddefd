"""Key metrics of ncu --set full captures (gpurun_out/prof2/fused_<cfg>.ncu-rep) into
profiles/<tag>_ncu_full_other.json: duration, DRAM bytes, issue activity, top stall reasons."""
import csv, io, json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1] if len(sys.argv) > 1 else "r1d"
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__inst_executed.avg.per_cycle_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "smsp__inst_executed.sum"]
out = {"how": "ncu --set full --clock-control none --import-source on -k regex:qrita_fused -s 3 -c 1 "
              "python bench.py --config <cfg> --steps 1 --warmup 3 --no-extras (cold caches, one launch)"}
for cfg in ("cfg1", "cfg3", "cfg4"):
    rep = os.path.join(ROOT, "gpurun_out", "prof2", f"fused_{cfg}.ncu-rep")
    if not os.path.exists(rep):
        continue
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(txt)))
    h, u, v = r[0], r[1], r[2]
    d = dict(zip(h, v)); un = dict(zip(h, u))
    m = {k: (float(d[k].replace(",", "")), un[k]) for k in KEYS if k in d}
    stalls = {k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""):
              float(d[k]) for k in h if k.startswith("smsp__average_warps_issue_stalled_") and
              k.endswith("_per_issue_active.ratio")}
    top = dict(sorted(stalls.items(), key=lambda t: -t[1])[:6])
    out[cfg] = {"kernel": d.get("Kernel Name", ""), "metrics": m, "top_stalls_per_issue": top}
json.dump(out, open(os.path.join(ROOT, "profiles", f"{tag}_ncu_full_other.json"), "w"), indent=1)
for c in ("cfg1", "cfg3", "cfg4"):
    if c in out:
        mm = out[c]["metrics"]
        print(c, mm.get("gpu__time_duration.sum"), mm.get("dram__bytes_read.sum"), out[c]["top_stalls_per_issue"])
