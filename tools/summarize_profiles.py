"""Turn the gpurun_out/prof captures of tools/round_profile.sh into the tracked summaries under
profiles/ (per-launch times and DRAM bytes per config, the --set full metrics of the dominant kernel,
and profiles/ncu_traffic.json, which bench.py reads for roofline.traffic)."""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "gpurun_out", "prof")
DST = os.path.join(ROOT, "profiles")
tag = sys.argv[1] if len(sys.argv) > 1 else "r1"


def launches(cfg):
    path = os.path.join(SRC, f"launches_{cfg}.csv")
    rows = [r for r in csv.reader(open(path)) if r and r[0] != "==PROF=="]
    hdr = next(i for i, r in enumerate(rows) if "Metric Name" in r)
    h = rows[hdr]
    out = {}
    for r in rows[hdr + 1:]:
        if len(r) < len(h):
            continue
        d = dict(zip(h, r))
        key = (d["ID"], d["Kernel Name"])
        out.setdefault(key, {})[d["Metric Name"]] = (float(d["Metric Value"].replace(",", "")), d["Metric Unit"])
    res = []
    for (lid, name), m in out.items():
        t, tu = m["gpu__time_duration.sum"]
        rd, ru = m["dram__bytes_read.sum"]
        wr, wu = m["dram__bytes_write.sum"]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9}
        tsc = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
        res.append({"id": int(lid), "kernel": name.split("(")[0], "us": t * tsc[tu],
                    "dram_read_bytes": rd * scale[ru], "dram_write_bytes": wr * scale[wu]})
    return res


summary = {}
for cfg in ("cfg2", "cfg4", "cfg3", "cfg1", "cfg5", "cfg2copy", "lmhead"):
    try:
        summary[cfg] = launches(cfg)
    except (OSError, StopIteration, KeyError) as e:
        print("skip", cfg, e)
with open(os.path.join(DST, f"{tag}_launches.json"), "w") as fh:
    json.dump({"how": "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                      "--clock-control none -k regex:qrita -s 3 -c 12 python bench.py --config <cfg> "
                      "--steps 3 --warmup 3 --no-extras (cold-cache, serialised: compare shares, not "
                      "absolutes)", "launches": summary}, fh, indent=1)

WANT = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed.avg.per_cycle_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__shared_mem_per_block_dynamic", "launch__shared_mem_per_block_static",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "lts__t_sectors_srcunit_tex_op_read.sum",
        "smsp__cycles_active.avg",
        "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
traffic = {}
for name, cfg, kern, how in (("fused_cfg2", "cfg2", "qrita_fused<float,3>", "-k regex:qrita_fused ... bench.py"),
                             ("topp16_cfg3", "cfg3", "qrita_topp16", "-k regex:qrita_topp16 ... bench.py --config cfg3"),
                             ("lmhead_gemm", "lmhead", "lmh_gemm<256,4>", "-k regex:lmh_gemm ... tools/lmh_prof.py")):
    rep = os.path.join(SRC, f"{name}.ncu-rep")
    if not os.path.exists(rep):
        continue
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h, units, v = rows[0], rows[1], rows[2]
    full = {w: [v[h.index(w)], units[h.index(w)]] for w in WANT if w in h}
    stalls = {k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""):
              float(v[i]) for i, k in enumerate(h) if k.startswith("smsp__average_warps_issue_stalled_") and
              k.endswith("_per_issue_active.ratio")}
    with open(os.path.join(DST, f"{tag}_ncu_full_{name}.json"), "w") as fh:
        hw = (f"ncu --set full --clock-control none --import-source on -k regex:lmh_gemm -s 1 -c 1 python "
              "tools/lmh_prof.py (one launch of the fused call's GEMM, B=256 V=128256 d=4096, cold caches)"
              if name == "lmhead_gemm" else
              f"ncu --set full --clock-control none --import-source on {how} --steps 1 --warmup 3 "
              "--no-extras (-s 3 -c 1: one launch, cold caches)")
        json.dump({"how": hw, "metrics": full,
                   "top_stalls_per_issue": dict(sorted(stalls.items(), key=lambda t: -t[1])[:8])}, fh, indent=1)
    rd = float(full["dram__bytes_read.sum"][0]) * SCALE[full["dram__bytes_read.sum"][1]]
    wr = float(full["dram__bytes_write.sum"][0]) * SCALE[full["dram__bytes_write.sum"][1]]
    traffic[cfg] = {"qrita_main_dram_bytes_per_launch": int(rd + wr), "kernel": kern,
                    "dram_read_bytes": int(rd), "dram_write_bytes": int(wr),
                    "source": f"profiles/{tag}_ncu_full_{name}.json (ncu --set full, dram__bytes_read.sum + "
                              "dram__bytes_write.sum)",
                    "note": "write bytes still in L2 (dirty) when the kernel ends are written back later "
                            "and not counted here"}
if traffic:
    with open(os.path.join(DST, "ncu_traffic.json"), "w") as fh:
        json.dump(traffic, fh, indent=1)
print(json.dumps({k: [(l["kernel"], round(l["us"], 1), round((l["dram_read_bytes"] + l["dram_write_bytes"]) / 1e6, 1)) for l in v] for k, v in summary.items()}, indent=0))
