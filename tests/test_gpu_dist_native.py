"""The C-ABI row-block power iteration (spmvb_dist_init/step/destroy over a
caller-owned NCCL communicator, SURVEY §8(b), and its overlapped-range form
spmvb_dist_init_ranges/step_ranges) against the torch.distributed driver
(dist.PowerIteration, its plain all-gatherv path): the same iterate, bit
for bit.  One process, a one-rank NCCL group (this project's boxes have
one GPU; tests/test_gpu_multi.py runs two ranks where two GPUs exist)."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, port_no, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port_no)
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    import paper_1805_11938_b200 as sp
    from paper_1805_11938_b200 import dist as spdist

    comm = dist.group.WORLD._get_backend(dev)._comm_ptr()
    import ctypes

    ver = ctypes.c_int()
    sp._lib.check(sp._lib.load().spmvb_dist_nccl_version(ctypes.byref(ver)))
    major, minor, patch = torch.cuda.nccl.version()
    # the library must drive the NCCL that made torch's communicator
    out["nccl"] = (ver.value, major * 10000 + minor * 100 + patch)
    r, c, v = sp.synth.rmat_triplets(14, 8, 77, dev)
    n = 1 << 14
    a = sp.canonicalize(r, c, v, n, n)
    x0 = sp.synth.uniform_vector(n, 5, device=dev)
    res = {}
    for tag, kw in [("csr5", dict(omega=32, sigma=16)), ("sell", dict(sell_c=32, sell_sigma=256)), ("hyb", {})]:
        m = sp.convert(tag, a, **kw)
        native = spdist.NativePowerIteration(sp.SpmvOperator(tag, m), [0, n], 0, 1, dev, x0, comm)
        plain = spdist.PowerIteration(lambda xv, o, s, tag=tag, m=m: sp.spmv(tag, m, xv, out=o, scale=s), [0, n], 0, 1,
                                      dev, x0)
        for _ in range(12):
            native.step()
            plain.step()
        torch.cuda.synchronize()
        res[tag] = (native.x.cpu().numpy().tobytes() == plain.x.cpu().numpy().tobytes(),
                    float(native.scale.item()) == float(plain.scale.item()), float(native.scale.item()))
        native.close()
        if tag in ("csr5", "sell"):  # the overlapped-range step (spmvb_dist_step_ranges)
            if tag == "csr5":
                tb, rb = m.range_plan(3)
                k = len(tb) - 1
                plan = [(int(rb[i]), int(rb[i + 1]) if i + 1 < k else m.n_rows, int(tb[i]), int(tb[i + 1]))
                        for i in range(k)][::-1]
                spans = [(p_[0], p_[1]) for p_ in plan]
            else:
                plan = m.range_plan(3)[::-1]
                spans = [(p_[6], p_[7]) for p_ in plan]
            rn = spdist.NativePowerIteration(
                sp.SpmvOperator(tag, m), [0, n], 0, 1, dev, x0, comm, ranges=spans,
                range_op=lambda k, xv, out, sc, tag=tag, m=m, plan=plan: sp.bind_range(tag, m, xv, out, plan[k], sc))
            for _ in range(12):
                rn.step()
            torch.cuda.synchronize()
            res[tag + "-ranges"] = (rn.x.cpu().numpy().tobytes() == plain.x.cpu().numpy().tobytes(),
                                   float(rn.scale.item()) == float(plain.scale.item()), float(rn.scale.item()))
            rn.close()
    out[0] = res
    dist.destroy_process_group()


def test_c_abi_power_iteration_matches_driver():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    out = mp.get_context("spawn").Manager().dict()
    mp.spawn(_worker, args=(_free_port(), out), nprocs=1, join=True)
    assert out["nccl"][0] == out["nccl"][1], out["nccl"]
    assert {"csr5-ranges", "sell-ranges"} <= set(out[0])
    for tag, (same_x, same_scale, scale) in out[0].items():
        assert same_x and same_scale, tag
        assert np.isfinite(scale) and scale > 0
