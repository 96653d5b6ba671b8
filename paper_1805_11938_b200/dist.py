"""1-D nnz-balanced row-block SpMV across GPUs.

One process per GPU (torch.distributed, NCCL over NVLink/NVSwitch).  Rank p
owns rows [r_p, r_{p+1}) of A (all columns) and a full copy of x.  Each
power-iteration step

    y_p = s * A_p x            (local SpMV, hand-written kernel, s deferred norm)
    ||y||^2 = sum_p ||y_p||^2  (1-double all-reduce)
    x <- all-gatherv(y_p)      (grouped P2P send/recv: true variable counts;
                                nnz-balanced shards differ ~100x in rows, so
                                an equal-count all-gather would pad ~3.5x)
    s <- 1 / ||y||

so x_{k+1} = A x_k / ||A x_k|| with the normalisation folded into the next
SpMV by linearity.  The local SpMV writes straight into this rank's slice
of the next x (no copy).  The same code runs over gloo with CPU tensors in
the tests (the local SpMV is injectable).

``exchange="p2p"`` does the all-gather with our own kernel over peer
memory instead of NCCL: x lives in symmetric memory mapped into every rank,
each finished row range is stored straight into the peers' next iterate
(overlapping the next range's SpMV), the per-rank ||y_p||^2 go into the
peers' norm slots, and one device-side barrier ends the step (no host
round trip, no NCCL).

``exchange="sparse"`` replaces the all-gatherv by the exchange of only the
x entries each shard's columns touch (§8(e): ~20% of the columns per shard
at C4, so ~4-5x less traffic): the column sets and the per-peer request
lists are exchanged once at setup; every step the owner packs the requested
entries of its y block (one gather kernel), grouped P2P moves them, and the
receiver unpacks them into its x (one scatter kernel).  Entries no local
column reads are left stale; ``gather_full()`` materialises the whole
iterate when it is wanted.
"""

from __future__ import annotations

import ctypes
import math
from typing import Callable

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from ._lib import LIB, check, ptr
from .formats import CsrMatrix

__all__ = ["nnz_balanced_bounds", "cost_balanced_bounds", "row_block", "PowerIteration", "NativePowerIteration",
           "GpuOps"]


def nnz_balanced_bounds(row_ptr, parts: int) -> np.ndarray:
    """Boundaries r_0 = 0 < ... < r_P = n: r_p = first row with
    ptr[r] >= ceil(p * nnz / P) (binary search on the CSR row pointer)."""
    p_host = row_ptr.cpu().numpy() if isinstance(row_ptr, torch.Tensor) else np.asarray(row_ptr)
    n = p_host.size - 1
    nnz = int(p_host[-1])
    targets = [-(-p * nnz // parts) for p in range(1, parts)]
    inner = np.searchsorted(p_host, targets, side="left") if parts > 1 else np.empty(0, np.int64)
    bounds = np.concatenate([[0], np.minimum(inner, n), [n]]).astype(np.int64)
    return np.maximum.accumulate(bounds)


def cost_balanced_bounds(row_ptr, parts: int, row_weight: float = 1.5) -> np.ndarray:
    """Row blocks balanced on nnz + row_weight * rows instead of nnz alone.

    A shard's SpMV time is not only its nonzeros: every row costs a y store
    (and the empty-row pass a ptr test), so on R-MAT the nnz-balanced shard
    holding the long tail of light rows is the slowest (C5, P = 8: 0.43 vs
    0.32 ms, profiles/r01_c5_shards.jsonl; fitting those shard times gives
    one row ~ 1.5 nonzeros).  r_p = first row whose prefix cost reaches
    p/P of the total."""
    p_host = row_ptr.cpu().numpy() if isinstance(row_ptr, torch.Tensor) else np.asarray(row_ptr)
    n = p_host.size - 1
    cost = p_host.astype(np.float64) + row_weight * np.arange(n + 1, dtype=np.float64)
    targets = [p * cost[-1] / parts for p in range(1, parts)]
    inner = np.searchsorted(cost, targets, side="left") if parts > 1 else np.empty(0, np.int64)
    bounds = np.concatenate([[0], np.minimum(inner, n), [n]]).astype(np.int64)
    return np.maximum.accumulate(bounds)


def row_block(csr: CsrMatrix, lo: int, hi: int) -> CsrMatrix:
    """Rows [lo, hi) of a CSR matrix as an independent CSR (all columns)."""
    a = int(csr.ptr[lo].item())
    b = int(csr.ptr[hi].item())
    p = (csr.ptr[lo : hi + 1] - a).contiguous()
    return CsrMatrix(hi - lo, csr.n_cols, p, csr.indices[a:b].clone(), csr.data[a:b].clone())


class GpuOps:
    """Device helpers of the power iteration (library kernels).  The gloo
    tests substitute CPU versions with the same contracts."""

    @staticmethod
    def sumsq(y: torch.Tensor, out: torch.Tensor) -> None:
        with torch.cuda.device(y.device):
            check(LIB.spmvb_sumsq(ptr(y), y.numel(), ptr(out), _lib.stream(y.device)))

    @staticmethod
    def inv_sqrt(sumsq: torch.Tensor, scale: torch.Tensor) -> None:
        with torch.cuda.device(sumsq.device):
            check(LIB.spmvb_inv_sqrt(ptr(sumsq), ptr(scale), _lib.stream(sumsq.device)))

    @staticmethod
    def bind_norm_scale(y: torch.Tensor, sumsq: torch.Tensor, scale: torch.Tensor):
        """A prepared ``sumsq = ||y||^2; scale = 1/||y||`` (one launch,
        spmvb_norm_scale) on these buffers, with its own workspace."""
        from .kernels import BoundCall

        ws = torch.zeros(int(LIB.spmvb_norm_ws_bytes()), dtype=torch.uint8, device=y.device)
        return BoundCall("spmvb_norm_scale", (ptr(y), y.numel(), ptr(ws), ptr(sumsq), ptr(scale)),
                         _lib.stream(y.device), keep=(y, sumsq, scale, ws))

    @staticmethod
    def column_set(cols: torch.Tensor, n_cols: int) -> torch.Tensor:
        """Sorted distinct column ids (int32) of ``cols``."""
        dev = cols.device
        cnt = ctypes.c_int64()
        with torch.cuda.device(dev):
            check(LIB.spmvb_column_set(ptr(cols), cols.numel(), n_cols, None, ctypes.byref(cnt), _lib.stream(dev)))
            out = torch.empty(cnt.value, dtype=torch.int32, device=dev)
            check(LIB.spmvb_column_set(ptr(cols), cols.numel(), n_cols, ptr(out), ctypes.byref(cnt),
                                       _lib.stream(dev)))
        return out

    @staticmethod
    def gather(src: torch.Tensor, base: int, idx: torch.Tensor, dst: torch.Tensor) -> None:
        with torch.cuda.device(src.device):
            check(LIB.spmvb_gather_f64(ptr(src), base, ptr(idx), idx.numel(), ptr(dst), _lib.stream(src.device)))

    @staticmethod
    def scatter(src: torch.Tensor, idx: torch.Tensor, dst: torch.Tensor) -> None:
        with torch.cuda.device(dst.device):
            check(LIB.spmvb_scatter_f64(ptr(src), ptr(idx), idx.numel(), ptr(dst), _lib.stream(dst.device)))


class PowerIteration:
    """Distributed power iteration over a row-block partition.

    ``local_spmv(x_full, out, scale)`` must write ``scale * A_p x_full`` into
    ``out`` (a view of this rank's slice of the next iterate).  ``exchange``
    is ``"allgatherv"`` (every rank holds the whole iterate) or ``"sparse"``
    (only the entries this shard's columns read; needs ``local_cols``, the
    shard's column indices).  ``ops`` supplies the device helpers (GpuOps by
    default; CPU substitutes in the gloo tests).

    Overlap (all-gatherv only): ``local_ranges`` lists this rank's row spans
    (local rows, in execution order, tiling [0, n_local)) and
    ``local_spmv_range(k, x_full, out, scale)`` computes span k into ``out``;
    each span is sent to the peers as soon as it is computed, so the
    exchange overlaps the remaining spans.  CSR5 shards
    use the row-aligned tile ranges of ``Csr5Matrix.range_plan`` with
    ``kernels.spmv_csr5_tiles``: bit-identical to the single-shot SpMV.
    """

    def __init__(self, local_spmv: Callable, bounds, rank: int, world: int, device: torch.device,
                 x0: torch.Tensor, group=None, ops=None, exchange: str = "allgatherv",
                 local_cols: torch.Tensor | None = None, local_ranges=None, local_spmv_range: Callable | None = None,
                 local_spmv_push: Callable | None = None, send_rows: int | None = None):
        if exchange not in ("allgatherv", "sparse", "p2p"):
            raise ValueError(f"unknown exchange {exchange!r}")
        if exchange == "p2p" and world > 1 and dist.get_backend(group) == dist.Backend.GLOO:
            raise ValueError("exchange='p2p' needs NCCL and peer-mapped GPUs, not gloo")
        self.local_spmv = local_spmv
        self.bounds = [int(b) for b in bounds]
        self.rank, self.world = rank, world
        self.group = group
        self.device = device
        self.ops = ops or GpuOps
        n = self.bounds[-1]
        self.x = x0.to(device=device, dtype=torch.float64).clone()
        self.x_next = torch.empty(n, dtype=torch.float64, device=device)
        self.sumsq = torch.zeros(1, dtype=torch.float64, device=device)
        self.scale = torch.ones(1, dtype=torch.float64, device=device)
        self.lo, self.hi = self.bounds[rank], self.bounds[rank + 1]
        # device tensors over a backend without a device transport (gloo):
        # every exchange is staged through a host copy of the iterate
        self._staged = (device.type == "cuda" and world > 1 and
                        dist.get_backend(self.group) == dist.Backend.GLOO)
        self._host = torch.empty(n if self._staged else 0, dtype=torch.float64, pin_memory=self._staged)
        # p2p also runs at world 1 (no peers: it exercises the buffers,
        # barrier and norm slots on one GPU)
        self.exchange = exchange if (world > 1 or exchange == "p2p") else "allgatherv"
        self._ranges_local = local_ranges
        self.local_spmv_range = local_spmv_range
        # exchange="p2p" with a fused kernel: local_spmv_push(x, out, scale,
        # peers, push_off) computes the shard and stores its rows into the
        # peers' next iterate in the same kernel (kernels.spmv_csr5_push)
        self.local_spmv_push = local_spmv_push
        if self.exchange == "p2p":
            self._plan_p2p(x0, n)
        if self.exchange == "sparse":
            if local_cols is None:
                raise ValueError("exchange='sparse' needs local_cols (the shard's column indices)")
            self._plan_sparse(local_cols, n)
        # prepared launches (single process, plain exchange, a local_spmv that
        # can bind, the library's ops): per x/x_next parity the SpMV and the
        # fused norm are bound once, so a step is two ctypes calls
        self._fast = None
        self._fast_ok = (world == 1 and self.exchange == "allgatherv" and device.type == "cuda"
                         and hasattr(local_spmv, "bind") and self.ops is GpuOps)
        # send_rows: this rank's rows past the first send_rows are empty, so
        # their entries of every iterate after the first are exactly 0 -- the
        # all-gatherv moves only each rank's leading send_rows rows and the
        # peers' empty tails are zeroed once (a degree-ordered shard: C5 has
        # 58 % empty rows)
        self._send_hi = list(self.bounds[1:])
        self._tails_pending = False
        if world > 1 and self.exchange == "allgatherv":
            mine = self.hi if send_rows is None else self.lo + min(max(int(send_rows), 0), self.hi - self.lo)
            allhi = [None] * world
            dist.all_gather_object(allhi, mine, group=self.group)
            self._send_hi = [int(v) for v in allhi]
            if self._send_hi != self.bounds[1:]:
                self._zero_remote_tails(self.x_next)
                self._tails_pending = True  # x (still x0) gets its remote tails zeroed after the first step
        self._spans = None
        if local_ranges is not None and world > 1 and self.exchange == "allgatherv":
            if local_spmv_range is None:
                raise ValueError("local_ranges needs local_spmv_range")
            spans = [(self.lo + int(a), self.lo + int(b)) for a, b in local_ranges]
            covered = sorted(spans)
            if covered and (covered[0][0] != self.lo or covered[-1][1] != self.hi or
                            any(covered[i][1] != covered[i + 1][0] for i in range(len(covered) - 1))):
                raise ValueError("local_ranges must tile this rank's rows")
            allspans = [None] * world
            dist.all_gather_object(allspans, spans, group=self.group)
            self._spans = allspans

    # ---- full exchange ---------------------------------------------------
    def _zero_remote_tails(self, buf: torch.Tensor) -> None:
        for p in range(self.world):
            if p != self.rank and self._send_hi[p] < self.bounds[p + 1]:
                buf[self._send_hi[p]:self.bounds[p + 1]].zero_()

    def _after_step(self) -> None:
        """Called after the swap: the first time, the old x0 buffer (now
        x_next) still holds x0 in the peers' empty tails; zero them."""
        if self._tails_pending:
            self._zero_remote_tails(self.x_next)
            self._tails_pending = False

    def _all_reduce_sumsq(self) -> None:
        if self._staged:
            s = self.sumsq.cpu()
            dist.all_reduce(s, group=self.group)
            self.sumsq.copy_(s)
        else:
            dist.all_reduce(self.sumsq, group=self.group)

    def _allgatherv(self, y_full: torch.Tensor) -> None:
        if self._staged:  # exchange host copies, then upload the peers' rows
            self._host[self.lo:self._send_hi[self.rank]].copy_(y_full[self.lo:self._send_hi[self.rank]])
            self._allgatherv_tensor(self._host)
            for p in range(self.world):
                lo, hi = self.bounds[p], self._send_hi[p]
                if p != self.rank and hi > lo:
                    y_full[lo:hi].copy_(self._host[lo:hi])
            return
        self._allgatherv_tensor(y_full)

    def _allgatherv_tensor(self, y_full: torch.Tensor) -> None:
        mine = y_full[self.lo : self._send_hi[self.rank]]
        ops = []
        for p in range(self.world):
            if p == self.rank:
                continue
            lo, hi = self.bounds[p], self._send_hi[p]
            if mine.numel():
                ops.append(dist.P2POp(dist.isend, mine, p, group=self.group))
            if hi > lo:
                ops.append(dist.P2POp(dist.irecv, y_full[lo:hi], p, group=self.group))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()

    # ---- sparse exchange -------------------------------------------------
    def _plan_sparse(self, local_cols: torch.Tensor, n: int) -> None:
        P, me = self.world, self.rank
        need = self.ops.column_set(local_cols.to(self.device), n)  # sorted, int32
        cuts = np.searchsorted(need.cpu().numpy(), self.bounds, side="left")
        recv_counts = [int(cuts[q + 1] - cuts[q]) if q != me else 0 for q in range(P)]
        # counts matrix: row p = what rank p receives from each owner
        xdev = torch.device("cpu") if self._staged else self.device  # where the collectives run
        mine = torch.tensor(recv_counts, dtype=torch.int64, device=xdev)
        allc = [torch.empty_like(mine) for _ in range(P)]
        dist.all_gather(allc, mine, group=self.group)
        send_counts = [int(allc[p][me].item()) if p != me else 0 for p in range(P)]
        # request lists: rank p tells owner q which of q's rows it reads
        send_idx = torch.empty(sum(send_counts), dtype=torch.int32, device=xdev)
        need_x = need.to(xdev)
        ops, s_off, r_off = [], [0], [0]
        for p in range(P):
            s_off.append(s_off[-1] + send_counts[p])
            r_off.append(r_off[-1] + recv_counts[p])
        for p in range(P):
            if p == me:
                continue
            if recv_counts[p]:
                ops.append(dist.P2POp(dist.isend, need_x[int(cuts[p]):int(cuts[p + 1])].contiguous(), p,
                                      group=self.group))
            if send_counts[p]:
                ops.append(dist.P2POp(dist.irecv, send_idx[s_off[p]:s_off[p + 1]], p, group=self.group))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        self._recv_idx = torch.cat([need[int(cuts[q]):int(cuts[q + 1])] for q in range(P) if q != me]) \
            if P > 1 else need[:0]
        self._send_idx = send_idx.to(self.device)
        self._send_counts, self._recv_counts = send_counts, recv_counts
        self._s_off, self._r_off = s_off, r_off
        self._send_buf = torch.empty(max(s_off[-1], 1), dtype=torch.float64, device=self.device)
        self._recv_buf = torch.empty(max(r_off[-1], 1), dtype=torch.float64, device=self.device)
        if self._staged:
            self._send_host = torch.empty(self._send_buf.numel(), dtype=torch.float64, pin_memory=True)
            self._recv_host = torch.empty(self._recv_buf.numel(), dtype=torch.float64, pin_memory=True)
        self.exchange_volume = {"send_entries": s_off[-1], "recv_entries": r_off[-1],
                                "allgatherv_recv_entries": n - (self.hi - self.lo)}

    def _sparse(self, y_full: torch.Tensor) -> None:
        mine = y_full[self.lo : self.hi]
        if self._send_idx.numel():
            self.ops.gather(mine, self.lo, self._send_idx, self._send_buf)
        send_buf, recv_buf = self._send_buf, self._recv_buf
        if self._staged:
            self._send_host.copy_(self._send_buf)
            send_buf, recv_buf = self._send_host, self._recv_host
        ops = []
        for p in range(self.world):
            if p == self.rank:
                continue
            if self._send_counts[p]:
                ops.append(dist.P2POp(dist.isend, send_buf[self._s_off[p]:self._s_off[p + 1]], p,
                                      group=self.group))
            if self._recv_counts[p]:
                ops.append(dist.P2POp(dist.irecv, recv_buf[self._r_off[p]:self._r_off[p + 1]], p,
                                      group=self.group))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        if self._staged:
            self._recv_buf.copy_(self._recv_host)
        if self._recv_idx.numel():
            self.ops.scatter(self._recv_buf, self._recv_idx, y_full)

    def _step_overlapped(self) -> None:
        """Row ranges in order; after each one its rows go to every peer
        (grouped P2P on the communicator's stream) while the next range
        computes.  Every rank walks the same range index k, so the k-th
        groups match pairwise."""
        me = self.rank
        out = self.x_next[self.lo : self.hi]
        # staged (gloo): each finished span is copied to the host and sent
        # from there; received spans are uploaded after the last wait
        buf = self._host if self._staged else self.x_next

        def clip(p, span):  # the part of a span that is sent (rows before the empty tail)
            return None if span is None else (span[0], max(span[0], min(span[1], self._send_hi[p])))

        reqs = []
        for k in range(max(len(sp) for sp in self._spans)):
            full = self._spans[me][k] if k < len(self._spans[me]) else None
            mine = clip(me, full)
            if full is not None:
                self.local_spmv_range(k, self.x, out, self.scale)
                if self._staged and mine[1] > mine[0]:
                    buf[mine[0]:mine[1]].copy_(self.x_next[mine[0]:mine[1]])
            ops = []
            for p in range(self.world):
                if p == me:
                    continue
                if mine is not None and mine[1] > mine[0]:
                    ops.append(dist.P2POp(dist.isend, buf[mine[0]:mine[1]], p, group=self.group))
                theirs = clip(p, self._spans[p][k] if k < len(self._spans[p]) else None)
                if theirs is not None and theirs[1] > theirs[0]:
                    ops.append(dist.P2POp(dist.irecv, buf[theirs[0]:theirs[1]], p, group=self.group))
            if ops:
                reqs.extend(dist.batch_isend_irecv(ops))
        self.ops.sumsq(out, self.sumsq)
        self._all_reduce_sumsq()
        for r in reqs:
            r.wait()
        if self._staged:
            for p in range(self.world):
                lo, hi = self.bounds[p], self._send_hi[p]
                if p != me and hi > lo:
                    self.x_next[lo:hi].copy_(buf[lo:hi])
        self.ops.inv_sqrt(self.sumsq, self.scale)
        self.x, self.x_next = self.x_next, self.x
        self._after_step()

    # ---- peer-memory exchange (our kernels over NVLink, no NCCL) ----------
    def _plan_p2p(self, x0: torch.Tensor, n: int) -> None:
        """x / x_next live in symmetric memory mapped into every rank; each
        step pushes this rank's rows straight into the peers' next iterate
        (spmvb_push_rows, one launch per finished row range on a side stream,
        overlapping the next range) and its ||y_p||^2 into their norm slots,
        then one device-side barrier ends the step.  Norm slots alternate
        between two halves by step parity, and a rank writes a peer's x only
        after the barrier that ends the peer's reads of it."""
        import torch.distributed._symmetric_memory as symm

        group = self.group if self.group is not None else dist.group.WORLD
        P, me, dev = self.world, self.rank, self.device
        self._bufs, self._handles, self._peer_ptrs = [], [], []
        for _ in range(2):
            b = symm.empty(max(n, 1), dtype=torch.float64, device=dev)
            h = symm.rendezvous(b, group)
            peers = [int(h.buffer_ptrs[q]) + int(h.offset) for q in range(P) if q != me]
            self._bufs.append(b)
            self._handles.append(h)
            self._peer_ptrs.append(torch.tensor(peers or [0], dtype=torch.int64, device=dev))
        if self._handles[0].buffer_ptrs[me] + self._handles[0].offset != self._bufs[0].data_ptr():
            raise RuntimeError("symmetric-memory peer addressing does not match the local buffer")
        self._sums = symm.empty(2 * P, dtype=torch.float64, device=dev)
        self._sums_h = symm.rendezvous(self._sums, group)
        self._sums_peers = torch.tensor(
            [int(self._sums_h.buffer_ptrs[q]) + int(self._sums_h.offset) for q in range(P) if q != me] or [0],
            dtype=torch.int64, device=dev)
        self._bufs[0][:n].copy_(x0.to(device=dev, dtype=torch.float64))
        self.x, self.x_next = self._bufs[0][:n], self._bufs[1][:n]
        self._cur = 0  # index of the buffer holding x
        self._parity = 0
        self._push_stream = torch.cuda.Stream(device=dev)

    def _push(self, buf_index: int, a: int, b: int) -> None:
        """Rows [a, b) (global) of buffer `buf_index` into the same rows of every peer's buffer."""
        if b <= a or self.world == 1:
            return
        src = self._bufs[buf_index][a:b]
        with torch.cuda.device(self.device):
            check(LIB.spmvb_push_rows(ptr(src), b - a, self._peer_ptrs[buf_index].data_ptr(), self.world - 1, a,
                                      _lib.stream(self.device)))

    def _step_p2p(self) -> None:
        nxt = 1 - self._cur
        out = self.x_next[self.lo : self.hi]
        main = torch.cuda.current_stream(self.device)
        if self.local_spmv_push is not None:
            peers = self._peer_ptrs[nxt] if self.world > 1 else self._peer_ptrs[nxt][:0]
            self.local_spmv_push(self.x, out, self.scale, peers, self.lo)
        elif self._ranges_local is not None and self.local_spmv_range is not None:
            for k, (a, b) in enumerate(self._ranges_local):
                self.local_spmv_range(k, self.x, out, self.scale)
                ev = torch.cuda.Event()
                ev.record(main)
                self._push_stream.wait_event(ev)
                with torch.cuda.stream(self._push_stream):
                    self._push(nxt, self.lo + a, self.lo + b)
            main.wait_stream(self._push_stream)
        else:
            self.local_spmv(self.x, out, self.scale)
            self._push(nxt, self.lo, self.hi)
        P, me = self.world, self.rank
        slot = self._parity * P + me
        self.ops.sumsq(out, self._sums[slot : slot + 1])
        if P > 1:
            with torch.cuda.device(self.device):
                check(LIB.spmvb_push_rows(ptr(self._sums[slot : slot + 1]), 1, self._sums_peers.data_ptr(), P - 1,
                                          slot, _lib.stream(self.device)))
        self._sums_h.barrier(channel=0)
        half = self._sums[self._parity * P : self._parity * P + P]
        with torch.cuda.device(self.device):
            check(LIB.spmvb_sum_inv_sqrt(ptr(half), P, ptr(self.sumsq), ptr(self.scale), _lib.stream(self.device)))
        self._parity ^= 1
        self._cur = nxt
        self.x, self.x_next = self.x_next, self.x

    def _fast_calls(self):
        """The bound (SpMV, norm) launches for the current x/x_next buffers
        and stream, bound on first use (at most a few sets are kept)."""
        key = (self.x.data_ptr(), self.x_next.data_ptr(), torch.cuda.current_stream(self.device).cuda_stream)
        f = self._fast
        if f is None or len(f) >= 4 and key not in f:
            f = self._fast = {}
        calls = f.get(key)
        if calls is None:
            out = self.x_next[self.lo : self.hi]
            calls = f[key] = (self.local_spmv.bind(self.x, out, self.scale),
                              GpuOps.bind_norm_scale(out, self.sumsq, self.scale))
        return calls

    def step(self) -> None:
        if self._fast_ok:
            spmv_call, norm_call = self._fast_calls()
            spmv_call()
            norm_call()
            self.x, self.x_next = self.x_next, self.x
            return
        if self.exchange == "p2p":
            self._step_p2p()
            return
        if self._spans is not None:
            self._step_overlapped()
            return
        out = self.x_next[self.lo : self.hi]
        self.local_spmv(self.x, out, self.scale)
        self.ops.sumsq(out, self.sumsq)
        if self.world > 1:
            self._all_reduce_sumsq()
            if self.exchange == "sparse":
                self._sparse(self.x_next)
            else:
                self._allgatherv(self.x_next)
        self.ops.inv_sqrt(self.sumsq, self.scale)
        self.x, self.x_next = self.x_next, self.x
        self._after_step()

    def gather_full(self) -> torch.Tensor:
        """The whole current iterate on every rank (one all-gatherv; a no-op
        for the full exchange)."""
        if self.world > 1 and self.exchange == "sparse":
            self._allgatherv(self.x)
        return self.x

    def run(self, steps: int, graph: bool | str = False) -> None:
        """``steps`` power-iteration steps, eagerly by default.

        ``graph=True`` (single process on CUDA, opt-in) captures two steps --
        one x/x_next ping-pong -- in a CUDA graph once and replays it, so
        launch-bound small matrices are not limited by host-side launch cost;
        an odd remainder step runs eagerly.  Capture contract: ``local_spmv``
        must not synchronise with the host (no host x/out, no ``.item()``)
        and must keep reading and writing the same buffers on every call
        (its matrix, scale and output pointers are frozen into the graph).
        Rebinding ``x``/``x_next`` is detected and re-captures; if capture
        fails the steps run eagerly (with a warning) and the iterate is left
        as eager steps would leave it.  ``graph="auto"`` times alternating
        rounds of eager steps and replays once (median of 3 each) and keeps
        the faster mode.  The p2p exchange (its symmetric-memory barrier is
        left eager) and multi-process runs never use the graph.  Iterates are
        bit-identical either way."""
        usable = self.world == 1 and self.device.type == "cuda" and self.exchange != "p2p"
        if graph == "auto":
            graph = getattr(self, "_graph_auto", None) if usable else False
            if graph is None:
                if steps < 16:
                    graph = False
                else:
                    steps = self._calibrate_graph(steps)
                    graph = self._graph_auto
        if not graph or not usable:
            for _ in range(steps):
                self.step()
            return
        bufs = (self.x.data_ptr(), self.x_next.data_ptr())
        g_bufs = getattr(self, "_graph_bufs", None)
        if getattr(self, "_graph", None) is not None and bufs not in (g_bufs, g_bufs[::-1]):
            self._graph = None  # buffers were rebound since the capture
        if getattr(self, "_graph", None) is None:
            if steps < 2:
                for _ in range(steps):
                    self.step()
                return
            side = torch.cuda.Stream(device=self.device)
            side.wait_stream(torch.cuda.current_stream(self.device))
            with torch.cuda.stream(side):  # two real steps warm the allocations
                self.step()
                self.step()
            torch.cuda.current_stream(self.device).wait_stream(side)
            steps -= 2
            g = torch.cuda.CUDAGraph()
            state = (self.x, self.x_next, self.sumsq.clone(), self.scale.clone())
            captured = (self.x.data_ptr(), self.x_next.data_ptr())
            err = self._capture(g)
            if err is not None:  # not capturable: restore the pre-capture state, run eagerly
                import warnings

                self.x, self.x_next = state[0], state[1]
                self.sumsq.copy_(state[2])
                self.scale.copy_(state[3])
                warnings.warn(f"PowerIteration: CUDA graph capture failed ({type(err).__name__}: {err}); "
                              "running eager steps", RuntimeWarning, stacklevel=2)
                self._graph = None
                for _ in range(steps):
                    self.step()
                return
            self._graph_bufs = captured  # the graph reads [0] as x
            self._graph = g
        if steps and self.x.data_ptr() != self._graph_bufs[0]:  # odd step count so far
            self.step()
            steps -= 1
        for _ in range(steps // 2):
            self._graph.replay()
        if steps % 2:
            self.step()

    def _capture(self, g) -> Exception | None:
        """Captures two steps into ``g`` on a side stream; returns the error
        if the steps could not be captured.  (Done by hand rather than with
        ``torch.cuda.graph``: when a capture is invalidated its exit raises
        before it restores the current stream and before the caching
        allocator stops routing allocations to the graph's pool.)"""
        dev = self.device
        pool = torch.cuda.graph_pool_handle()
        side = torch.cuda.Stream(device=dev)
        side.wait_stream(torch.cuda.current_stream(dev))
        err = None
        with torch.cuda.stream(side):
            g.capture_begin(pool=pool)
            try:
                self.step()
                self.step()
            except Exception as exc:
                err = exc
            try:
                g.capture_end()
            except Exception as exc:
                err = err or exc
                torch._C._cuda_endAllocateToPool(dev.index if dev.index is not None else torch.cuda.current_device(),
                                                 pool)
        torch.cuda.current_stream(dev).wait_stream(side)
        if err is not None:
            torch.cuda.synchronize(dev)
        return err

    def _calibrate_graph(self, steps: int) -> int:
        """Runs 16 of ``steps``: the capture (2 warm-up steps, 2 replays),
        then three alternating rounds of 2 timed eager steps and 1 timed
        replay (2 steps); keeps the mode with the smaller median in
        ``_graph_auto`` and drops the graph when eager wins.  Returns the
        steps left."""
        main = torch.cuda.current_stream(self.device)
        self._graph = None
        self.run(4, graph=True)
        if getattr(self, "_graph", None) is None:  # capture failed: eager
            self._graph_auto = False
            return steps - 4
        if self.x.data_ptr() != self._graph_bufs[0]:
            self.step()
            steps -= 1
        ev = []
        for _ in range(3):
            e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            e[0].record(main)
            self.step()
            self.step()
            e[1].record(main)
            self._graph.replay()
            e[2].record(main)
            ev.append(e)
        torch.cuda.synchronize(self.device)
        eager = sorted(e[0].elapsed_time(e[1]) for e in ev)[1]
        replay = sorted(e[1].elapsed_time(e[2]) for e in ev)[1]
        self._graph_auto = replay < eager
        if not self._graph_auto:
            self._graph = None  # release the graph and its private pool
        return steps - 16

    def normalized(self) -> torch.Tensor:
        """The unit-norm iterate ``scale * x`` (``x`` holds the last SpMV
        output; its normalisation is deferred into the next SpMV)."""
        return self.x * self.scale

    def eigenvalue_estimate(self) -> float:
        """||A x_k|| for the current normalised iterate (1/scale)."""
        s = float(self.scale.item())
        return 1.0 / s if s > 0 else math.nan


class NativePowerIteration:
    """The row-block power iteration through the C ABI's ``spmvb_dist_*``
    (a caller-owned NCCL communicator): one ctypes call per
    step, NCCL issued from C, no per-op Python work.  ``local_op`` binds the
    shard's SpMV (``kernels.SpmvOperator`` or ``relabel.RelabelledMatrix``);
    ``comm_ptr`` is the ``ncclComm_t`` address (from torch:
    ``group._get_backend(device)._comm_ptr()``).  With ``ranges`` (this
    rank's local row spans in execution order) and ``range_op(k, x, out,
    scale)`` returning a prepared launch of span k (``kernels.bind_range``), each
    span's rows go to the peers while the next span computes
    (``spmvb_dist_step_ranges``); the spans of all ranks are exchanged once
    here over ``group``.  Same iterate as ``PowerIteration``'s all-gatherv
    path, bit for bit."""

    _CB = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                           ctypes.c_void_p)
    _RCB = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                            ctypes.c_void_p, ctypes.c_void_p)

    def __init__(self, local_op, bounds, rank: int, world: int, device: torch.device, x0: torch.Tensor,
                 comm_ptr: int, ranges=None, range_op: Callable | None = None, group=None,
                 send_rows: int | None = None):
        self.bounds = [int(b) for b in bounds]
        self.rank, self.world, self.device = rank, world, device
        n = self.bounds[-1]
        lo, hi = self.bounds[rank], self.bounds[rank + 1]
        self.x = x0.to(device=device, dtype=torch.float64).clone()
        self.x_next = torch.empty(n, dtype=torch.float64, device=device)
        self.sumsq = torch.zeros(1, dtype=torch.float64, device=device)
        self.scale = torch.ones(1, dtype=torch.float64, device=device)
        pairs = ((self.x, self.x_next), (self.x_next, self.x))
        self._ranged = ranges is not None
        # send_rows as in PowerIteration: only each rank's leading send_rows
        # rows travel; the peers' empty tails are zeroed once
        limit = hi - lo if send_rows is None else min(max(int(send_rows), 0), hi - lo)
        if self._ranged:
            if range_op is None:
                raise ValueError("ranges need range_op")
            spans = [(int(a), int(b)) for a, b in ranges]
            sent = [(a, max(a, min(b, limit))) for a, b in spans]
            allspans = [None] * world
            if world > 1:
                dist.all_gather_object(allspans, (sent, lo + limit), group=group)
            else:
                allspans = [(sent, lo + limit)]
            self._send_hi = [int(h_) for _, h_ in allspans]
            K = max(len(sp_) for sp_, _ in allspans)
            flat = []
            for sp_, _ in allspans:
                sp_ = sp_ + [(0, 0)] * (K - len(sp_))
                flat += [v for ab in sp_ for v in ab]
            self._calls = {(int(a.data_ptr()), k): range_op(k, a, b[lo:hi], self.scale) for a, b in pairs
                           for k in range(len(spans))}

            def local(ctx, k, x, y, scale, stream):
                call = self._calls.get((int(x), int(k)))
                if call is None:  # past this rank's own ranges
                    return 0
                try:
                    call()
                    return 0
                except Exception:  # reported through the status code
                    return _lib.SPMVB_INTERNAL

            self._cb = self._RCB(local)
            b_arr = (ctypes.c_int64 * len(self.bounds))(*self.bounds)
            s_arr = (ctypes.c_int64 * len(flat))(*flat)
            h = ctypes.c_void_p()
            check(LIB.spmvb_dist_init_ranges(ctypes.c_void_p(comm_ptr), rank, world, b_arr, K, s_arr,
                                             ctypes.byref(h)))
        else:
            if send_rows is not None:
                raise ValueError("send_rows needs ranges (spmvb_dist_step_ranges)")
            self._send_hi = list(self.bounds[1:])
            # the SpMV of each parity, bound once; the callback picks it by x
            self._calls = {int(a.data_ptr()): local_op.bind(a, b[lo:hi], self.scale) for a, b in pairs}

            def local(ctx, x, y, scale, stream):
                try:
                    self._calls[int(x)]()
                    return 0
                except Exception:  # reported through the status code
                    return _lib.SPMVB_INTERNAL

            self._cb = self._CB(local)  # keep the callback alive with the object
            b_arr = (ctypes.c_int64 * len(self.bounds))(*self.bounds)
            h = ctypes.c_void_p()
            check(LIB.spmvb_dist_init(ctypes.c_void_p(comm_ptr), rank, world, b_arr, ctypes.byref(h)))
        self._h = h
        self._tails_pending = self._send_hi != self.bounds[1:]
        if self._tails_pending:
            self._zero_tails(self.x_next)
        self.exchange = "allgatherv"
        self.driver = "c-abi spmvb_dist_step" + ("_ranges" if self._ranged else "")

    def _zero_tails(self, buf: torch.Tensor) -> None:
        for p in range(self.world):
            if p != self.rank and self._send_hi[p] < self.bounds[p + 1]:
                buf[self._send_hi[p]:self.bounds[p + 1]].zero_()

    def step(self) -> None:
        fn = LIB.spmvb_dist_step_ranges if self._ranged else LIB.spmvb_dist_step
        with torch.cuda.device(self.device):
            check(fn(self._h, ctypes.cast(self._cb, ctypes.c_void_p), None, ptr(self.x), ptr(self.x_next),
                     ptr(self.sumsq), ptr(self.scale), _lib.stream(self.device)))
        self.x, self.x_next = self.x_next, self.x
        if self._tails_pending:  # the old x0 buffer still holds x0 in the peers' empty tails
            self._zero_tails(self.x_next)
            self._tails_pending = False

    def eigenvalue_estimate(self) -> float:
        s = float(self.scale.item())
        return 1.0 / s if s > 0 else math.nan

    def close(self) -> None:
        if getattr(self, "_h", None):
            check(LIB.spmvb_dist_destroy(self._h))
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
