"""SURVEY.md §8c crossing-margin audit: for every top-p row of cfg1-cfg5, the relative distance
between p and the two exactly rounded prefix sums that straddle the nucleus crossing
(oracle.crossing_margin).  A row below 1e-13 is "ulp-sensitive": its kept set could depend on the
last bit of exp() / the normaliser, where this build (CUDA exp, exactly rounded normaliser) and the
reference (numpy AVX-512 exp, pairwise sum) may differ.  Writes profiles/margin_audit.json.

    python tools/margin_audit.py [--procs 8]
"""
import argparse
import concurrent.futures as cf
import json
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle.qrita_oracle import crossing_margin  # noqa: E402
from oracle.synth import config_inputs  # noqa: E402

THRESH = 1e-13
_X = {}


def _init(name):
    _X["x"], _X["k"], _X["p"], _ = config_inputs(name)


def _rows(idx):
    x, k, p = _X["x"], _X["k"], _X["p"]
    return [(int(i), crossing_margin(x[i], int(k[i]), float(p[i]))) for i in idx]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--procs", type=int, default=os.cpu_count() or 1)
    args = ap.parse_args()
    report = {"threshold": THRESH, "definition": "min(|fsum(prefix_L) - p|, |p - fsum(prefix_{L-1})|) / p over "
              "the oracle's probabilities (oracle.py:70-89); SURVEY.md 8c", "configs": {}}
    for name in ("cfg1", "cfg2", "cfg3", "cfg4", "cfg5"):
        x, k, p, _ = config_inputs(name)
        rows = np.nonzero(p < 1.0)[0]
        chunks = np.array_split(rows, max(1, min(len(rows), 4 * args.procs)))
        with cf.ProcessPoolExecutor(args.procs, initializer=_init, initargs=(name,)) as ex:
            res = [r for part in ex.map(_rows, chunks) for r in part]
        m = np.array([v for _, v in res])
        finite = m[np.isfinite(m)]
        report["configs"][name] = {
            "rows": int(x.shape[0]), "topp_rows": int(len(rows)),
            "ulp_sensitive_rows": int((m < THRESH).sum()),
            "min_margin": float(finite.min()) if finite.size else math.inf,
            "p10_margin": float(np.percentile(finite, 10)) if finite.size else math.inf,
            "median_margin": float(np.median(finite)) if finite.size else math.inf,
            "rows_below_1e-10": int((m < 1e-10).sum()),
            "min_rows": [int(i) for i, v in sorted(res, key=lambda t: t[1])[:3]],
        }
        print(name, report["configs"][name], flush=True)
    with open(os.path.join(ROOT, "profiles", "margin_audit.json"), "w") as fh:
        json.dump(report, fh, indent=1)


if __name__ == "__main__":
    main()
