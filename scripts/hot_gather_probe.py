"""Gather-rate probe with the hot head of the degree-ordered x in shared memory
(scripts/hot_gather_probe.cu): G gathers/s over the degree-ordered C4 / C5
column indices in CSR order (row-consecutive lanes) and in SELL-32 order
(lane per row), for hot = 0 .. 24576 columns and 512 / 1024 threads per SM.

    python scripts/hot_gather_probe.py [C4 C5]
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import bench  # noqa: E402
import paper_1805_11938_b200 as sp  # noqa: E402
from paper_1805_11938_b200 import _lib, synth  # noqa: E402
from paper_1805_11938_b200.relabel import DegreeOrder  # noqa: E402


def build():
    so = ROOT / "scripts" / "libhotprobe.so"
    src = ROOT / "scripts" / "hot_gather_probe.cu"
    if not so.exists() or so.stat().st_mtime < src.stat().st_mtime:
        subprocess.check_call(["nvcc", "-O3", "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler",
                               "-fPIC", "-o", str(so), str(src)])
    lib = ctypes.CDLL(str(so))
    lib.hot_probe.restype = ctypes.c_int
    lib.hot_probe.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_int,
                              ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
    lib.dot_probe.restype = ctypes.c_int
    lib.dot_probe.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int,
                              ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
    return lib


def timed(fn, reps=5):
    for _ in range(2):
        fn()
    best = 1e9
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        best = min(best, a.elapsed_time(b))
    return best * 1e-3


def main():
    lib = build()
    dev = torch.device("cuda", 0)
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    stream = torch.cuda.current_stream(dev).cuda_stream
    for cfg in (sys.argv[1:] or ["C4", "C5"]):
        w = bench.WORKLOADS[cfg]
        csr = sp.to_csr(bench.build_workload(sp, synth, w, dev))
        x = synth.uniform_vector(csr.n_cols, w["x_seed"], device=dev)
        order = DegreeOrder(csr, key="row")
        csr, x = order.matrix(csr), order.to_new(x)
        sell = sp.convert("sell", csr, sell_c=32, sell_sigma=0, max_cells=1 << 34)
        streams = {"csr-order": csr.indices, "sell-order": sell.flat_indices}
        if os.environ.get("HOT_PROBE_MASKED"):
            # every index folded into [0, 16384): hot = 16384 is then all LDS,
            # mode 2 all L1-resident LDG -- the two paths' own ceilings
            streams = {"csr-order&16383": csr.indices & 16383, "uniform-random<16384": torch.randint(
                0, 16384, (csr.nnz,), dtype=torch.int32, device=dev)}
        part = torch.empty(sms * 8 * 1024, dtype=torch.float64, device=dev)
        for name, idx in streams.items():
            n = idx.numel()
            base = timed(lambda: _lib.check(_lib.load().spmvb_gather_probe(x.data_ptr(), idx.data_ptr(), n,
                                                                            part.data_ptr(), stream)))
            print(f"{cfg} {name:10s} n {n:>10d}  library probe (148x8 CTAs of 256, U16): {n / base / 1e9:7.1f} G/s "
                  f"({base * 1e6:8.1f} us)", flush=True)
            if os.environ.get("HOT_PROBE_DOT"):
                # the SpMV's traffic without its row structure: sum val[i] * x[idx[i]]
                val = torch.rand(n, dtype=torch.float64, device=dev)
                for threads, blocks in ((1024, sms), (512, 2 * sms), (256, 5 * sms), (256, 8 * sms)):
                    for u in (4, 8):
                        def rund():
                            rc = lib.dot_probe(x.data_ptr(), idx.data_ptr(), val.data_ptr(), n, threads, blocks, u,
                                               part.data_ptr(), stream)
                            assert rc == 0, rc
                        t = timed(rund)
                        print(f"{cfg} {name:10s} flat dot product, {blocks} CTAs of {threads}, U {u}: "
                              f"{n / t / 1e9:7.1f} G/s ({t * 1e6:8.1f} us)", flush=True)
                del val
                continue
            ref = None
            for threads in (512, 1024):
                for u in (4, 8):
                    for mode, hots in ((2, (0,)), (0, (4096, 8192, 12288, 16384, 24576)),
                                       (1, (8192, 16384))):
                        for hot in hots:
                            def run():
                                rc = lib.hot_probe(x.data_ptr(), idx.data_ptr(), n, hot, threads, sms, mode, u,
                                                   part.data_ptr(), stream)
                                assert rc == 0, rc
                            t = timed(run)
                            s = float(part[: sms * threads].sum().item())
                            if ref is None:
                                ref = s
                            ok = abs(s - ref) <= 1e-9 * abs(ref)
                            print(f"{cfg} {name:10s} threads {threads:4d} U {u:2d} mode {mode} hot {hot:5d}: "
                                  f"{n / t / 1e9:7.1f} G/s ({t * 1e6:8.1f} us){'' if ok else '  SUM MISMATCH'}",
                                  flush=True)
        del csr, sell, x, part
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
