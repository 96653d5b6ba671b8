"""DRAM traffic per SpMV for the kernels bench.py reports (roofline.traffic).

Run under ncu with profiling off at start; every target's ONE timed SpMV is
bracketed by cudaProfilerStart/Stop, so the capture holds exactly the
kernels of those SpMVs, in target order:

    ncu --set full --import-source on --clock-control none --profile-from-start off \
        -o gpurun_out/ncu_traffic python scripts/ncu_traffic.py --plan gpurun_out/ncu_traffic_plan.json
    python scripts/ncu_traffic.py --parse gpurun_out/ncu_traffic.ncu-rep --plan gpurun_out/ncu_traffic_plan.json

The parse step (here, no GPU) sums dram__bytes_read.sum + dram__bytes_write.sum
over each target's kernels and writes profiles/ncu_traffic.json keyed
"<config>/<variant>[-relabel]/n1" as bench.py looks them up.
"""

from __future__ import annotations

import argparse
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

TARGETS = [
    "C5/csr5-w32s16-relabel", "C5/sell-c32s0-relabel", "C5/sell-c32s8192-relabel", "C5/csr5-w32s8-relabel", "C5/hyb-relabel",
    "C5/csr-relabel", "C5/csr5-w32s16", "C5/csr", "C5/hyb", "C5/sell-c32s8192",
    "C4/csr5-w32s16-relabel", "C4/csr5-w32s8-relabel", "C4/sell-c32s0-relabel", "C4/sell-c32s8192-relabel", "C4/hyb-relabel",
    "C4/csr-relabel", "C4/csr5-w32s16", "C4/csr", "C4/hyb",
    "C3/ell", "C3/hyb", "C3/sell-c32s1024", "C3/csr5-w32s16",
    "C2/ell", "C2/hyb", "C2/csr5-w32s16",
    "C1/ell", "C1/hyb", "C1/csr",
]


def parse_variant(v):
    relabel = v.endswith("-relabel")
    v = v[: -len("-relabel")] if relabel else v
    if v.startswith("csr5-"):
        w, s = v[len("csr5-w"):].split("s")
        return "csr5", dict(omega=int(w), sigma=int(s)), relabel
    if v.startswith("sell-"):
        c, s = v[len("sell-c"):].split("s")
        return "sell", dict(sell_c=int(c), sell_sigma=int(s), max_cells=1 << 34), relabel
    return v, ({"max_cells": 1 << 34} if v == "hyb" else {}), relabel


def capture(plan_path, targets):
    import torch

    import bench
    import paper_1805_11938_b200 as sp
    from paper_1805_11938_b200 import _lib, synth
    from paper_1805_11938_b200.relabel import RelabelledMatrix

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    plan = []
    cache = {}
    for t in targets:
        cfg, var = t.split("/")
        w = bench.WORKLOADS[cfg]
        if cfg not in cache:
            cache.clear()
            torch.cuda.empty_cache()
            a = bench.build_workload(sp, synth, w, dev)
            cache[cfg] = (sp.to_csr(a), synth.uniform_vector(a.n_cols, w["x_seed"], device=dev))
            del a
        csr, x = cache[cfg]
        tag, kw, relabel = parse_variant(var)
        if relabel:
            rm = RelabelledMatrix(tag, csr, **kw)
            xv = rm.order.to_new(x)
            fn = lambda: rm.spmv(xv)  # noqa: E731
        else:
            m = sp.convert(tag, csr, **kw)
            fn = lambda: sp.spmv(tag, m, x)  # noqa: E731
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        n0 = _lib.load().spmvb_launch_count()
        torch.cuda.cudart().cudaProfilerStart()
        fn()
        torch.cuda.synchronize()
        torch.cuda.cudart().cudaProfilerStop()
        plan.append({"target": t, "kernels": int(_lib.load().spmvb_launch_count() - n0)})
        print(plan[-1], flush=True)
        del fn
    Path(plan_path).write_text(json.dumps(plan, indent=1))


def parse(rep, plan_path, out_path):
    plan = json.loads(Path(plan_path).read_text())
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                          "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head = rows[0]
    units = rows[1]
    data = rows[2:]
    col = {name: head.index(name) for name in ("Kernel Name", "dram__bytes_read.sum", "dram__bytes_write.sum",
                                                "gpu__time_duration.sum")}
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
             "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0, "B": 1, "KB": 1e3, "MB": 1e6,
             "GB": 1e9}

    def val(r, name):
        return float(r[col[name]].replace(",", "")) * scale[units[col[name]]]

    try:  # merge into the existing table (targets captured in other runs stay)
        out = json.loads(Path(out_path).read_text())
    except (OSError, ValueError):
        out = {}
    out["_source"] = ("ncu --set full --clock-control none (cache control all: cold caches), one SpMV per target "
                      "= all its kernels; dram__bytes_read.sum + dram__bytes_write.sum; scripts/ncu_traffic.py")
    detail = {}
    i = 0
    for p in plan:
        ks = data[i:i + p["kernels"]]
        i += p["kernels"]
        tb = sum(val(r, "dram__bytes_read.sum") + val(r, "dram__bytes_write.sum") for r in ks)
        out[f"{p['target']}/n1"] = int(tb)
        detail[p["target"]] = [{"kernel": r[col["Kernel Name"]][:80], "us": val(r, "gpu__time_duration.sum") * 1e6,
                                "read_MB": val(r, "dram__bytes_read.sum") / 1e6,
                                "write_MB": val(r, "dram__bytes_write.sum") / 1e6} for r in ks]
    if i != len(data):
        raise SystemExit(f"plan covers {i} kernels, capture holds {len(data)}")
    Path(out_path).write_text(json.dumps(out, indent=1) + "\n")
    print(json.dumps(detail, indent=1))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--plan", required=True)
    ap.add_argument("--parse", default=None, help="an .ncu-rep to read (no GPU needed)")
    ap.add_argument("--out", default=str(ROOT / "profiles" / "ncu_traffic.json"))
    ap.add_argument("--targets", default=",".join(TARGETS))
    args = ap.parse_args()
    if args.parse:
        parse(args.parse, args.plan, args.out)
    else:
        capture(args.plan, args.targets.split(","))


if __name__ == "__main__":
    main()
