"""Benchmark: exact Top-k + Top-p truncation on B200 (BASELINE.json metric, config cfg2).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config cfg2]

One "step" = one truncation pass over one synthetic batch: cfg2 = Llama-3 vocab V=128256, B=256
fp32 rows, per-row k ~ U{1..1024}, p ~ U[0.5, 0.99] (same law and seeds as the
reference's synth_batch).  Inputs are resident in HBM; L2 (126 MB) is flushed between timed steps
by writing a 256 MB buffer; every step is timed with CUDA events on the launching stream.

Multi-GPU (one process per GPU): under torchrun every rank reads RANK / WORLD_SIZE; without torchrun,
``--gpus N`` (N > 1) re-launches itself under torch.distributed.run with N ranks (and fails loudly if
fewer than N GPUs are visible).  Rows shard by contiguous blocks, no collective on the data path:
  cfg2 — weak scaling: every rank truncates its own 256-row batch (per-GPU work fixed);
  cfg4 — strong scaling: the one B=1024 x V=262144 batch is split into contiguous B/N row blocks
         (paper_2602_01518_b200.sharded.rank_rows), the BASELINE's row-sharded config.
The job time is the max over ranks of the event-timed steps (synchronised start: barrier + sync).

Extra keys beside the driver contract: roofline (dominant kernel qrita_fused vs the measured HBM
peak), cpu_baseline (the reference's own run_batch on the host cores, persistent process pool),
torch_sort_baseline (serving-stack torch.sort recipe on the same GPU), e2e (pinned host buffers
through the public API, copies inside), e2e_run_batch (the reference's entry point run_batch on
numpy arrays, everything inside).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "rows/sec and HBM GB/s (% of roofline) for Top-k+Top-p at B=256, V=128k"
FALLBACK_HBM_GBS = 6650.0


def _normal_rows(seed: int, rows: int, vocab: int, lo: int, hi: int, chunk: int = 64) -> np.ndarray:
    """Rows [lo, hi) of default_rng(seed).normal(0, 1, (rows, vocab)).astype(f32), generated in row
    chunks so a rank holds only its own block (the draws are sequential: same values as one call)."""
    rng = np.random.default_rng(seed)
    out = np.empty((hi - lo, vocab), dtype=np.float32)
    r = 0
    while r < hi:
        n = min(chunk, hi - r)
        blk = rng.normal(0.0, 1.0, (n, vocab))
        a, b = max(r, lo), min(r + n, hi)
        if b > a:
            out[a - lo:b - lo] = blk[a - r:b - r]
        r += n
    return out


def workload(name: str, rank: int = 0, world: int = 1):
    """Synthetic inputs of this rank (float32 matrix, k, p, dtype label, description, global rows,
    scaling) — same laws / seeds as SURVEY.md §8d."""
    if name == "cfg2":  # weak scaling: every rank owns a full 256-row batch of its own
        x = np.random.default_rng(1 + 1000 * rank).normal(0.0, 1.0, (256, 128256)).astype(np.float32)
        r = np.random.default_rng(42 + rank)
        return x, r.integers(1, 1025, 256).astype(np.int64), r.uniform(0.5, 0.99, 256), "f32", \
            "cfg2: Llama-3 V=128256, B=256 fp32, k~U{1..1024}, p~U[0.5,0.99]", 256 * world, "weak"
    if name == "cfg2h":  # first 128 rows of cfg2 (one row tail per SM)
        x, k, p, dt, *_ = workload("cfg2")
        return x[:128].copy(), k[:128].copy(), p[:128].copy(), dt, "cfg2 rows 0-127", 128 * world, "weak"
    if name == "cfg2copy":  # streaming floor: same matrix, k = V and p = 1 (passthrough copy)
        x = np.random.default_rng(1).normal(0.0, 1.0, (256, 128256)).astype(np.float32)
        return x, np.full(256, 128256, np.int64), np.full(256, 1.0), "f32", "cfg2 matrix, passthrough", \
            256 * world, "weak"
    if name == "cfg2k":  # top-k only
        x = np.random.default_rng(1).normal(0.0, 1.0, (256, 128256)).astype(np.float32)
        r = np.random.default_rng(42)
        return x, r.integers(1, 1025, 256).astype(np.int64), np.full(256, 1.0), "f32", "cfg2 top-k only", \
            256 * world, "weak"
    if name == "cfg1":
        x = np.random.default_rng(0).normal(0.0, 1.0, (1, 32000)).astype(np.float32)
        return x, np.full(1, 50, np.int64), np.full(1, 0.9), "f32", "cfg1: V=32000, B=1 fp32, k=50, p=0.9", \
            world, "weak"
    if name == "cfg3":
        x = np.random.default_rng(3).normal(0.0, 1.0, (64, 151936)).astype(np.float32)
        neg = x < 0
        x[neg] = np.round(4.0 * x[neg]) / 4.0
        return x, np.full(64, 151936, np.int64), np.full(64, 0.95), "bf16", \
            "cfg3: Qwen2 V=151936, B=64 bf16 quantised tail, top-p 0.95", 64 * world, "weak"
    if name == "cfg4":  # strong scaling: contiguous B/N row blocks of the one 1024-row batch
        from paper_2602_01518_b200.sharded import rank_rows
        lo, hi = rank_rows(1024, rank, world)
        x = _normal_rows(4, 1024, 262144, lo, hi)
        r = np.random.default_rng(44)
        k, p = r.integers(1, 1025, 1024).astype(np.int64), r.uniform(0.5, 0.99, 1024)
        return x, k[lo:hi].copy(), p[lo:hi].copy(), "f32", \
            f"cfg4: Gemma V=262144, B=1024 fp32, k~U{{1..1024}}, p~U[0.5,0.99]; rows {lo}-{hi - 1} of 1024 " \
            f"on this rank", 1024, "strong"
    raise ValueError(name)


def measured_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback"


def ncu_traffic(config: str):
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as fh:
            return json.load(fh).get(config, {}).get("qrita_main_dram_bytes_per_launch")
    except Exception:
        return None


class ClockSampler:
    """Samples SM clock and throttle reasons through NVML while the timed region runs."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown", 0x1: "gpu_idle"}

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                mask = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if mask & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.0005)

    def __enter__(self):
        if self.nv is not None:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv is not None:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                    "samples": 0}
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def cpu_model() -> str:
    """The host CPU model (lscpu's 'Model name'), for the CPU baseline's record."""
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_reference(x, k, p, procs: int, steps: int, warmup: int, kind: str = "run_batch"):
    """The reference's own CPU path on the host cores: sigmatop.run_batch (or sort_select) over
    contiguous row chunks in a persistent pool of `procs` processes (oracle/cpu_baseline.py; pool
    start-up outside the timed steps).  Falls back to the oracle port when the reference is not
    installed in baseline/_ref.  Returns (rows/s, per-step seconds, record)."""
    from oracle.cpu_baseline import CpuPool, reference_available
    ok, why = reference_available()
    pool_kind = kind if ok else "port"
    rows = np.arange(x.shape[0])
    with CpuPool(x, k, p, procs, pool_kind) as pool:
        for _ in range(warmup):
            pool.run(rows)
        walls = [pool.run(rows) for _ in range(steps)]
        startup = pool.startup_s
    med = statistics.median(walls)
    what = {"run_batch": "sigmatop.run_batch (pkg/src/sigmatop/engine.py:82-113, EngineConfig(threads=1) "
                         "per process)",
            "sort_select": "sigmatop.engine.sort_select (engine.py:183-205, the sort-based definition)",
            "port": "oracle/qrita_oracle.py (numpy restatement of oracle.py:70-89; reference not installed: "
                    + str(why) + ")"}[pool_kind]
    rec = {"value": x.shape[0] / med, "unit": "rows/s", "cores": procs,
           "kind": "reference" if ok else "port", "cpu_model": cpu_model(), "host_cores": os.cpu_count(),
           "sample": f"all {x.shape[0]} rows of the workload per step through {what}, contiguous row "
                     f"chunks over {procs} persistent worker processes; median of {steps} steps after "
                     f"{warmup} warm-up; pool start-up {startup:.2f}s excluded",
           "step_s": walls}
    return x.shape[0] / med, walls, rec


def run_reference(args):
    """--impl reference: the reference's own CPU implementation (sigmatop.run_batch from baseline/_ref)
    on all host cores, on the same workload as our arm.  Under torchrun only rank 0 runs."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    if rank != 0:
        return
    if args.config == "lmhead":
        print(json.dumps({"impl": "reference", "unavailable": "the reference has no LM-head producer "
                          "(SURVEY.md 8(f) rank 3); compare with this line's unfused_ms instead"}), flush=True)
        return
    x, k, p, dtype, desc, total_rows, scaling = workload(args.config, 0, 1)
    if args.config == "cfg4":  # the whole 1024-row batch (the CPU path is not sharded over GPUs)
        x, k, p, dtype, desc, total_rows, scaling = workload(args.config, 0, 1)
    procs = os.cpu_count() or 1
    value, walls, rec = cpu_reference(x, k, p, procs, args.steps, min(args.warmup, 2))
    rec["value"] = value
    line = {
        "metric": METRIC, "value": value, "unit": "rows/s", "impl": "reference",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * statistics.median(walls), "higher_is_better": True, "scaling": scaling,
        "vs_baseline": None, "dtype": dtype, "data": "synthetic",
        "config": {"workload": desc, "batch": int(x.shape[0]), "vocab": int(x.shape[1])},
        "cpu_baseline": rec,
        "e2e": {"value": value, "unit": "rows/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _spawn_ranks(args) -> int:
    """bench.py --gpus N outside torchrun: re-launch under torch.distributed.run with N ranks."""
    import socket
    import subprocess

    import torch
    have = torch.cuda.device_count()
    if have < args.gpus:
        print(json.dumps({"error": f"--gpus {args.gpus} needs {args.gpus} visible GPUs, found {have}"}),
              flush=True)
        sys.stderr.write(f"bench.py: --gpus {args.gpus} needs {args.gpus} visible GPUs, found {have}\n")
        return 2
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip e2e / torch.sort / cpu legs")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    if args.gpus < 1:
        ap.error("--gpus must be >= 1")
    if args.impl == "reference":
        return run_reference(args)
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(_spawn_ranks(args))

    import torch
    import torch.distributed as dist

    import ctypes

    import paper_2602_01518_b200 as Q
    from paper_2602_01518_b200 import _native as N
    from paper_2602_01518_b200.sortsel import torch_sort_topk_topp

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        sys.stderr.write(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}\n")
        sys.exit(2)
    if world > 1:
        if torch.cuda.device_count() <= local:
            sys.stderr.write(f"bench.py: rank {rank} needs GPU {local}, {torch.cuda.device_count()} visible\n")
            sys.exit(2)
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)

    if args.config == "cfg5":
        return bench_tp(args, rank, world, dev)
    if args.config == "lmhead":
        return bench_lmhead(args, rank, world, dev)
    x_np, k_np, p_np, dtype, desc, total_rows, scaling = workload(args.config, rank, world)
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    x = torch.from_numpy(x_np).to(dev).to(tdt)
    k = torch.from_numpy(k_np).to(dev)
    p = torch.from_numpy(p_np).to(dev)
    out = torch.empty_like(x)
    b, v = x.shape
    esize = x.element_size()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    flush_sink = torch.empty(1, dtype=torch.float32, device=dev)

    def l2_flush():
        # write 256 MB (> 126 MB L2), then read it back: the read evicts the dirty flush lines, so their
        # write-back happens here (untimed) and not inside the next timed step
        flush.zero_()
        torch.sum(flush, dim=0, keepdim=True, out=flush_sink)
    st = torch.cuda.current_stream(dev)

    def step(ev0, ev1):
        ev0.record(st)
        Q.topk_topp(x, k, p, out=out, check=False)
        ev1.record(st)

    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(args.steps)]
    for _ in range(args.warmup):
        l2_flush()
        Q.topk_topp(x, k, p, out=out, check=True)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            l2_flush()  # L2 flush between timed steps (not timed)
            step(*evs[i])
        torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    step_ms = [a.elapsed_time(c) for a, c in evs]
    total_ms = sum(step_ms)
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    value = total_rows * args.steps / (total_ms / 1e3)   # rows of ALL ranks / max-over-ranks time
    ms_per_step = total_ms / args.steps

    # per-kernel times (profiling iterations, untimed above): the events serialise the launches, so
    # prep / stream / tail are each measured alone on the launching stream
    prof = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(max(5, min(args.steps, 20)))]
    for e0, e1, e2, e3 in prof:
        l2_flush()
        e0.record(st)
        Q.topk_topp(x, k, p, out=out, check=False, prep_event=e1, stream_event=e2)
        e3.record(st)
    torch.cuda.synchronize(dev)
    prep_ms = statistics.mean(a.elapsed_time(bb) for a, bb, _, _ in prof)
    stream_ms = statistics.mean(bb.elapsed_time(c) for _, bb, c, _ in prof)
    tail_ms = statistics.mean(c.elapsed_time(d) for _, _, c, d in prof)

    # roofline of the dominant kernel: qrita_fused (one launch per step) reads and writes the [B, V]
    # matrix once; its time is the e1 -> e2 interval of the profiling iterations above
    kind = Q.ops.pipeline_kind(x)
    alg_bytes = b * v * esize * 2
    achieved = alg_bytes / (stream_ms / 1e3) / 1e9
    peak, peak_kind = measured_peak()
    traffic = ncu_traffic(args.config)
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic,
                "peak_source": peak_kind,
                "kernel": ("qrita_topp16 + qrita_fused (top-p-only bf16 rows in qrita_topp16, the fused "
                           "kernel skips them)" if dtype == "bf16" and kind == "fused" else
                           "qrita_fused" if kind == "fused" else "qrita_stream"),
                "kernel_ms": stream_ms, "alg_bytes_per_launch": alg_bytes,
                "alg_bytes_note": "B*V*sizeof(dtype) read + the same written (SURVEY.md 8d)",
                "step_frac": alg_bytes / (ms_per_step / 1e3) / 1e9 / peak}
    if traffic:
        # DRAM-side rate: bytes ncu saw move during the kernel / its time (write-back of output still
        # dirty in L2 at kernel end happens afterwards and is not in `traffic`)
        roofline["dram_side_gbs"] = traffic / (stream_ms / 1e3) / 1e9
        roofline["dram_side_frac"] = roofline["dram_side_gbs"] / peak
    if kind == "staged":
        roofline.update({"prep_ms": prep_ms, "tail_ms_serialised": tail_ms})
    launches_per_step = (2 if dtype == "bf16" else 1) if kind == "fused" else 3
    # passes over the logits per row (qrita_row_metrics.row_passes): 1 = read once from HBM
    met = Q.ops.metrics_buffer(b, dev)
    Q.topk_topp(x, k, p, out=out, metrics=met, check=True)
    passes = [m["row_passes"] for m in Q.ops.decode_metrics(met)]

    line = {
        "metric": METRIC, "value": value, "unit": "rows/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": scaling, "vs_baseline": None, "dtype": dtype, "data": "synthetic",
        "config": {"workload": desc if world == 1 else desc.replace(" on this rank", " on rank 0"),
                   "batch": total_rows, "vocab": v, "rows_per_gpu": b,
                   "l2": "flushed between steps (256 MB write + read-back, untimed)",
                   "parallelism": f"row-sharded x{world} ({scaling} scaling: "
                                  + ("each rank its own batch" if scaling == "weak" else "contiguous B/N row blocks")
                                  + "), no collective"},
        "hbm_gbs": alg_bytes / (ms_per_step / 1e3) / 1e9,
        "roofline": roofline,
        "clocks": clk.summary(),
        "gpu_launches": launches_per_step * args.steps,
        "passes_over_logits": {"mean": sum(passes) / len(passes), "max": max(passes)},
        "pipeline": kind,
    }

    if not args.no_extras:
        # torch.sort serving-stack baseline on the same GPU (not exact; throughput yardstick)
        for _ in range(3):
            torch_sort_topk_topp(x.float(), k, p)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ts = []
        for _ in range(max(5, min(args.steps, 20))):
            l2_flush()
            e0.record(st)
            torch_sort_topk_topp(x, k, p)
            e1.record(st)
            torch.cuda.synchronize(dev)
            ts.append(e0.elapsed_time(e1))
        sort_val = b / (statistics.mean(ts) / 1e3)
        line["torch_sort_baseline"] = {"value": sort_val, "unit": "rows/s",
                                       "ms_per_step": statistics.mean(ts), "exact": False,
                                       "ours_over_sort": (b / (ms_per_step / 1e3)) / sort_val}
        # index-only output (qrita_topk_topp_idx, out = NULL): kept columns instead of masked logits,
        # same selection; algorithmic bytes V*s read + kept*4 written per row
        kidx = torch.empty((b, v), dtype=torch.int32, device=dev)
        kcnt = torch.empty((b,), dtype=torch.int32, device=dev)
        for _ in range(3):
            Q.topk_topp_indices(x, k, p, kept_idx=kidx, kept_count=kcnt, check=True)
        ti = []
        for _ in range(max(5, min(args.steps, 20))):
            l2_flush()
            e0.record(st)
            Q.topk_topp_indices(x, k, p, kept_idx=kidx, kept_count=kcnt, check=False)
            e1.record(st)
            torch.cuda.synchronize(dev)
            ti.append(e0.elapsed_time(e1))
        idx_bytes = b * v * esize + int(kcnt.sum().item()) * 4
        idx_ms = statistics.mean(ti)
        line["index_only"] = {"value": b / (idx_ms / 1e3), "unit": "rows/s", "ms_per_step": idx_ms,
                              "alg_bytes": idx_bytes, "achieved_gbs": idx_bytes / (idx_ms / 1e3) / 1e9,
                              "frac": idx_bytes / (idx_ms / 1e3) / 1e9 / peak,
                              "api": "topk_topp_indices (qrita_topk_topp_idx, no masked logits)"}
        # e2e through the public API with HOST buffers: Q.topk_topp on pinned host tensors copies row
        # chunks in, truncates and copies them back with both transfer directions overlapped with the
        # kernels (native qrita_topk_topp_host); status-checked; the copies are inside the timed region
        x_host = torch.from_numpy(x_np).to(tdt).pin_memory()
        k_host, p_host = torch.from_numpy(k_np), torch.from_numpy(p_np)
        o_host = torch.empty_like(x_host).pin_memory()
        e2e_steps = max(3, min(args.steps, 10))
        tt = []
        for i in range(e2e_steps + 2):
            torch.cuda.synchronize(dev)
            e0.record(st)
            Q.topk_topp(x_host, k_host, p_host, out=o_host, check=True)
            e1.record(st)
            torch.cuda.synchronize(dev)
            if i >= 2:
                tt.append(e0.elapsed_time(e1))
        h2d = x_host.numel() * x_host.element_size() + b * 16
        # what the host pipeline downloads: the masked rows, or (sparse form, every row top-k with
        # k <= 4096) each row's kept columns + counts, the host building the masked rows; plus the
        # status words
        d2h = int(N.load().qrita_host_download_bytes(b, v, 0 if dtype == "f32" else 1,
                                                     ctypes.c_void_p(k_host.data_ptr()),
                                                     ctypes.c_void_p(x_host.data_ptr()),
                                                     ctypes.c_void_p(o_host.data_ptr()))) + b * 8
        e2e_ms = sharded_max(statistics.mean(tt), world, dev)
        line["e2e"] = {"value": total_rows / (e2e_ms / 1e3), "unit": "rows/s", "h2d_bytes_per_step": h2d,
                       "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms,
                       "api": "paper_2602_01518_b200.topk_topp(pinned host tensors)"}
        # e2e through the reference's own entry point: run_batch(LogitBatch(numpy), TruncTargets(numpy))
        # -> numpy float32 outputs + BatchReport (pageable host memory, validation, metrics report);
        # host wall clock around the call (it returns with the result in host memory)
        if dtype == "f32":
            batch = Q.LogitBatch(x_np)
            targets = Q.TruncTargets(k_np, p_np)
            cfg = Q.EngineConfig()
            rb = []
            for i in range(e2e_steps + 2):
                t0 = time.perf_counter()
                outs, rep = Q.run_batch(batch, targets, cfg)
                if i >= 2:
                    rb.append(time.perf_counter() - t0)
            rb_ms = sharded_max(1e3 * statistics.mean(rb), world, dev)
            line["e2e_run_batch"] = {"value": total_rows / (rb_ms / 1e3), "unit": "rows/s", "ms_per_step": rb_ms,
                                     "h2d_bytes_per_step": x_np.nbytes + b * 16,
                                     "d2h_bytes_per_step": x_np.nbytes + b * 48,
                                     "api": "paper_2602_01518_b200.run_batch(LogitBatch(numpy), TruncTargets(numpy), "
                                            "EngineConfig()) -> (numpy outputs, BatchReport)"}
        if rank == 0 and world == 1 and not args.no_cpu_baseline:
            procs = os.cpu_count() or 1
            x_cpu = x.float().cpu().numpy() if dtype == "bf16" else x_np  # the values the GPU sees
            val, walls, rec = cpu_reference(x_cpu, k_np, p_np, procs, steps=2, warmup=1)
            line["cpu_baseline"] = rec
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(line), flush=True)


def bench_tp(args, rank: int, world: int, dev):
    """cfg5: vocab-sharded (TP = world) truncation of B=128 x V=262144 fp32, every rank its column
    shard; per-row partials through a library-owned NCCL communicator (qrita_topk_topp_tp).  Job time
    = max over ranks of the event-timed calls."""
    import torch
    import torch.distributed as dist

    from paper_2602_01518_b200.tp import NcclComm, shard_bounds, topk_topp_tp
    b, v = 128, 262144
    x_np = np.random.default_rng(5).normal(0.0, 1.0, (b, v)).astype(np.float32)
    r = np.random.default_rng(55)
    k_np, p_np = r.integers(1, 1025, b).astype(np.int64), r.uniform(0.5, 0.99, b)
    bounds = shard_bounds(v, world)
    shard = torch.from_numpy(x_np[:, bounds[rank]:bounds[rank + 1]].copy()).to(dev)
    k, p = torch.from_numpy(k_np).to(dev), torch.from_numpy(p_np).to(dev)
    out = torch.empty_like(shard)
    comm = NcclComm()
    kcap = int(k_np.max())
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    st = torch.cuda.current_stream(dev)

    def call():
        topk_topp_tp(shard, k, p, vocab_offset=bounds[rank], vocab_size=v, comm=comm, k_cap=kcap, out=out,
                     topp_only_rows=False)
    flush_sink = torch.empty(1, dtype=torch.float32, device=dev)

    def l2_flush():  # as in the single-GPU arm: write 256 MB, read it back (clean eviction)
        flush.zero_()
        torch.sum(flush, dim=0, keepdim=True, out=flush_sink)
    for _ in range(args.warmup):
        l2_flush()
        call()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(args.steps)]
    with ClockSampler(dev.index) as clk:
        for e0, e1 in evs:
            l2_flush()
            if world > 1:
                dist.barrier()   # synchronised start of every step
            e0.record(st)
            call()
            e1.record(st)
        torch.cuda.synchronize(dev)
    ms = statistics.mean(a.elapsed_time(c) for a, c in evs)
    ms = sharded_max(ms, world, dev)
    peak, peak_kind = measured_peak()
    alg = b * (bounds[rank + 1] - bounds[rank]) * 4 * 2
    kmax = min(kcap, bounds[rank + 1] - bounds[rank])
    line = {
        "metric": METRIC, "value": b / (ms / 1e3), "unit": "rows/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"cfg5: vocab-sharded TP={world}, B=128 x V=262144 fp32, k~U{{1..1024}}, "
                               f"p~U[0.5,0.99]; shard [128, {bounds[1] - bounds[0]}] per rank",
                   "batch": b, "vocab": v, "l2": "flushed between steps (256 MB write + read-back, untimed)",
                   "parallelism": f"tp{world} (vocab shards, NCCL partials)"},
        "roofline": {"bound": "hbm", "achieved": alg / (ms / 1e3) / 1e9, "peak": peak, "unit": "GB/s",
                     "frac": alg / (ms / 1e3) / 1e9 / peak, "traffic": None, "peak_source": peak_kind,
                     "kernel": "whole qrita_topk_topp_tp call (kernels + collectives)",
                     "alg_bytes_per_launch": alg},
        "exchange_bytes_per_row_per_rank": 8 * kmax + 4,
        "clocks": clk.summary(),
        "gpu_launches": 5 * args.steps,  # prep, local fused, sorted pack, merge resolve, write (+ NCCL all-gather)
    }
    comm.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(line), flush=True)


def bench_lmhead(args, rank: int, world: int, dev):
    """LM head (Llama-3-8B shape: d=4096, V=128256, B=256 rows per GPU) + exact
    Top-k/Top-p, fused (qrita_lmhead_topk_topp: tcgen05 GEMM with the streaming pass in its epilogue).
    Random-init bf16 weights and hidden states; every rank its own replica (weak scaling).  The
    roofline is the tensor-core one (2*B*V*d flops per call) against the measured bf16 peak; the
    unfused pipeline (same GEMM, then topk_topp_indices on the logits) is reported beside it."""
    import torch
    import torch.distributed as dist

    from paper_2602_01518_b200.lmhead import lm_head_logits, lm_head_topk_topp
    import paper_2602_01518_b200 as Q
    b, v, d = 256, 128256, 4096
    g = torch.Generator(device="cpu").manual_seed(17 + rank)
    h = torch.randn(b, d, generator=g).to(torch.bfloat16).to(dev)
    w = (torch.randn(v, d, generator=g) / d ** 0.5).to(torch.bfloat16).to(dev)
    r = np.random.default_rng(2 + rank)
    k = torch.from_numpy(r.integers(1, 1025, b).astype(np.int64)).to(dev)
    p = torch.from_numpy(r.uniform(0.5, 0.99, b)).to(dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    sink = torch.empty(1, dtype=torch.float32, device=dev)
    st = torch.cuda.current_stream(dev)

    def l2_flush():
        flush.zero_()
        torch.sum(flush, dim=0, keepdim=True, out=sink)

    def timed(fn, steps):
        for _ in range(2):  # untimed: library handles / first-call setup
            fn()
        evs = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(steps)]
        for e0, e1 in evs:
            l2_flush()
            e0.record(st)
            fn()
            e1.record(st)
        torch.cuda.synchronize(dev)
        return statistics.mean(a.elapsed_time(c) for a, c in evs)

    fused = lambda: lm_head_topk_topp(h, w, k, p)
    logits = torch.empty(b, v, dtype=torch.float32, device=dev)
    unfused = lambda: Q.topk_topp_indices(lm_head_logits(h, w, out=logits), k, p)
    for _ in range(args.warmup):
        l2_flush()
        fused()
        unfused()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    with ClockSampler(dev.index) as clk:
        ms = timed(fused, args.steps)
    ms = sharded_max(ms, world, dev)
    ms_unfused = sharded_max(timed(unfused, max(3, args.steps // 2)), world, dev)
    ms_gemm = sharded_max(timed(lambda: lm_head_logits(h, w, out=logits), max(3, args.steps // 2)), world, dev)
    ms_cublas = sharded_max(timed(lambda: h @ w.T, max(3, args.steps // 2)), world, dev)
    # end to end: hidden states from pinned host memory in; the kept columns (compact lists,
    # k_cap = 1024), their logits and the counts back to the host
    h_host = h.cpu().pin_memory()
    kcap = 1024
    kidx_host = torch.empty(b, kcap, dtype=torch.int32).pin_memory()
    kval_host = torch.empty(b, kcap, dtype=torch.float32).pin_memory()
    kc_host = torch.empty(b, dtype=torch.int32).pin_memory()

    def e2e():
        hd = h_host.to(dev, non_blocking=True)
        lg, kidx, kc = lm_head_topk_topp(hd, w, k, p, k_cap=kcap)
        kval = torch.gather(lg, 1, kidx.clamp(0, v - 1).long())  # entries past kc[r] are ignored
        kidx_host.copy_(kidx, non_blocking=True)
        kval_host.copy_(kval, non_blocking=True)
        kc_host.copy_(kc, non_blocking=True)
    ms_e2e = sharded_max(timed(e2e, max(3, args.steps // 2)), world, dev)
    flops = 2.0 * b * v * d
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            peak, kind = float(json.load(fh)["bf16_tflops"]), "measured"
    except Exception:
        peak, kind = 2250.0, "fallback (nominal dense bf16)"
    line = {
        "metric": "rows/sec for LM head + Top-k+Top-p (fused), B=256, V=128k, d=4096", "value": world * b / (ms / 1e3),
        "unit": "rows/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16 (fp32 accumulate)",
        "data": "synthetic (random-init bf16 LM-head weights and hidden states)",
        "config": {"workload": "lmhead: Llama-3-8B LM head (d=4096, V=128256), B=256 rows per GPU, "
                               "k~U{1..1024}, p~U[0.5,0.99]", "batch": b, "vocab": v, "hidden": d,
                   "l2": "flushed between steps (256 MB write + read-back, untimed)"},
        "roofline": {"bound": "tensor", "achieved": flops / (ms / 1e3) / 1e12, "peak": peak, "unit": "TFLOP/s",
                     "frac": flops / (ms / 1e3) / 1e12 / peak, "traffic": None, "peak_source": kind,
                     "kernel": "whole qrita_lmhead_topk_topp call (GEMM + epilogue + row tails)"},
        "unfused_ms": ms_unfused, "gemm_only_ms": ms_gemm, "cublas_bf16_matmul_ms": ms_cublas,
        "e2e": {"value": world * b / (ms_e2e / 1e3), "unit": "rows/s", "h2d_bytes_per_step": b * d * 2,
                "d2h_bytes_per_step": b * kcap * 8 + b * 4, "ms_per_step": ms_e2e,
                "api": "lm_head_topk_topp(hidden from pinned host memory, k_cap=1024) -> kept columns, their "
                       "logits and counts to pinned host memory"},
        "clocks": clk.summary(),
        "gpu_launches": 2 * args.steps,  # lmh_gemm, qrita_tail (plus a counter memset)
    }
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(line), flush=True)


def sharded_max(ms: float, world: int, dev) -> float:
    """Max over ranks of a per-rank time (the job time)."""
    if world == 1:
        return ms
    import torch
    import torch.distributed as dist
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


if __name__ == "__main__":
    main()
