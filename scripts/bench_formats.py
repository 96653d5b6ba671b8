"""Per-config, per-format SpMV table on one B200 (kernel-only device time).

    python scripts/bench_formats.py [--configs C1,C2,C3,C4] [--reps 20] [--out profiles/r01_formats.jsonl]

For every BASELINE.json config C1-C4 and every format (reference default
parameters AND the GPU-tuned ones) it times y = A x with CUDA events, flushing
L2 (a 512 MB read) before every rep so the number is an HBM number; it also
reports the hot (no-flush) time.  Algorithmic bytes = the reference byte
model (harness.spmv_bytes); GFLOP/s = 2 nnz / t.  Each record also holds the
conversion time and a parity check against dense_spmv_oracle on the device
(max |y - y_seq| / (|A||x|)).
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import paper_1805_11938_b200 as sp  # noqa: E402
from paper_1805_11938_b200 import synth  # noqa: E402

VARIANTS = [
    ("csr", "default", {}),
    ("csr5", "default w4 s16", dict(omega=4, sigma=16)),
    ("csr5", "tuned w32 s16", dict(omega=32, sigma=16)),
    ("ell", "default", {}),
    ("sell", "default C4 s0", dict(sell_c=4, sell_sigma=0)),
    ("sell", "tuned C32 s0", dict(sell_c=32, sell_sigma=0, max_cells=1 << 34)),
    ("sell", "tuned C32 s1024", dict(sell_c=32, sell_sigma=1024, max_cells=1 << 34)),
    ("hyb", "default", {}),
]


def build(name):
    if name in ("C1", "C2", "C3"):
        return synth.host_coo(name)
    cfg = synth.CONFIGS[name]
    return synth.rmat_coo(cfg["scale"], cfg["edge_factor"], cfg["seed"])


def timed(fn, reps, flush):
    """Median device time of fn(); all reps are enqueued before one sync so
    the host runs ahead (the 512 MB flush in front of each rep hides the
    host-side launch cost).  The flush READS 512 MB, so L2 is left holding
    clean foreign lines: a write flush would leave ~126 MB of dirty lines
    whose write-back would be charged to the kernel."""
    evs = []
    torch.cuda.synchronize()
    for _ in range(reps):
        if flush is not None:
            flush.sum()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        evs.append((s, e))
    torch.cuda.synchronize()
    times = sorted(s.elapsed_time(e) / 1e3 for s, e in evs)
    return times[len(times) // 2]


def graph_time(fn, reps):
    """Hot per-call device time from one CUDA graph holding `reps` calls
    (no host launch gaps); None if capture is not possible."""
    try:
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            fn()
        torch.cuda.current_stream().wait_stream(s)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(reps):
                fn()
        g.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        b.synchronize()
        return a.elapsed_time(b) / 1e3 / reps
    except RuntimeError:
        return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C1,C2,C3,C4")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] if (ROOT / "MEASURED_PEAKS.json").exists() else 6650.0
    flush = torch.zeros(64 << 20, dtype=torch.float64, device="cuda")  # 512 MB, read before each cold rep
    out = open(args.out, "w") if args.out else None
    for name in args.configs.split(","):
        a = build(name)
        x = synth.uniform_vector(a.n_cols, 11)
        y = torch.empty(a.n_rows, dtype=torch.float64, device="cuda")
        ref = sp.dense_spmv_oracle(a, x)
        absA = sp.CooMatrix(a.n_rows, a.n_cols, a.row, a.col, a.data.abs())
        bound = sp.dense_spmv_oracle(absA, x.abs())
        for tag, label, kw in VARIANTS:
            rec = {"config": name, "format": tag, "variant": label, "n": a.n_rows, "nnz": a.nnz}
            try:
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                m = sp.convert(tag, a, **kw)
                torch.cuda.synchronize()
                rec["convert_ms"] = (time.perf_counter() - t0) * 1e3
            except sp.ConversionError as exc:
                rec["error"] = str(exc)[:100]
                print(json.dumps(rec), flush=True)
                if out:
                    out.write(json.dumps(rec) + "\n")
                continue
            fn = lambda: sp.spmv(tag, m, x, out=y)  # noqa: E731
            for _ in range(3):
                fn()
            cold = timed(fn, args.reps, flush)
            hot = graph_time(fn, args.reps) or timed(fn, args.reps, None)
            b = sp.spmv_bytes(tag, m)
            err = ((y - ref).abs() / bound.clamp_min(1e-300)).max().item() if a.n_rows else 0.0
            ok = bool(((y - ref).abs() <= 1e-12 * bound).all().item())
            rec.update(cold_us=cold * 1e6, hot_us=hot * 1e6, gflops=2 * a.nnz / cold / 1e9,
                       gbs_model=b / cold / 1e9, frac=b / cold / 1e9 / peak, hot_gflops=2 * a.nnz / hot / 1e9,
                       bytes_model=b, max_rel_err=err, within_tol=ok)
            print(json.dumps(rec), flush=True)
            if out:
                out.write(json.dumps(rec) + "\n")
            del m
        del a
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
