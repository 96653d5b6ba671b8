"""Host cost of one eager power-iteration step (C1-C3, the launch-bound
configs): the generic path (a Python local_spmv calling spmv(); sumsq and
inv_sqrt launched separately) against the prepared path (SpmvOperator:
the SpMV and the fused norm bound once per buffer parity), and the
device time per step for both and for graph replay.

    python scripts/dispatch_probe.py > profiles/r02_dispatch_probe.txt

host us/step: wall time of 2000 enqueued steps / 2000, measured while the
GPU is still busy with earlier ones (the launch queue never fills on these
sizes because each step's kernels finish faster than the host enqueues).
"""

from __future__ import annotations

import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import paper_1805_11938_b200 as sp  # noqa: E402
from paper_1805_11938_b200 import dist as spdist, synth  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    for name in ("C1", "C2", "C3"):
        a = synth.host_coo(name, device=dev)
        m = sp.to_ell(a)
        x0 = synth.uniform_vector(a.n_cols, 1, device=dev)
        variants = {
            "generic": lambda: spdist.PowerIteration(lambda x, o, s: sp.spmv("ell", m, x, out=o, scale=s),
                                                     [0, a.n_rows], 0, 1, dev, x0),
            "prepared": lambda: spdist.PowerIteration(sp.SpmvOperator("ell", m), [0, a.n_rows], 0, 1, dev, x0),
        }
        for label, make in variants.items():
            pi = make()
            for _ in range(20):
                pi.step()
            torch.cuda.synchronize()
            n = 2000
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev0.record()
            t0 = time.perf_counter()
            for _ in range(n):
                pi.step()
            t_host = time.perf_counter() - t0
            ev1.record()
            ev1.synchronize()
            t_dev = ev0.elapsed_time(ev1) / 1e3
            print(f"{name} ell {label:8s}: host {t_host / n * 1e6:6.2f} us/step, device {t_dev / n * 1e6:6.2f} "
                  f"us/step (eager)", flush=True)
            if label == "prepared":
                pi.run(4, graph=True)
                torch.cuda.synchronize()
                ev0.record()
                pi.run(n, graph=True)
                ev1.record()
                ev1.synchronize()
                print(f"{name} ell {label:8s}: device {ev0.elapsed_time(ev1) / 1e3 / n * 1e6:6.2f} us/step "
                      f"(graph replay)", flush=True)
            del pi
        del a, m
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
