"""Padding of the SELL-32 sigma 0 slices on the degree-ordered layout: cells
(32 x width per slice) against stored nonzeros, for all slices, for the wide
slices (width > wide_cols(), summed by k_sell_wide_part) and for the hub
slices (more than SELL_HUB_PIECES pieces): C4 whole, C5 whole, C5 dealt
shard 0 of 2 / 4 / 8.

    python scripts/sell_padding_probe.py > profiles/r02_sell_padding_probe.txt
"""

from __future__ import annotations

import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import bench  # noqa: E402
import paper_1805_11938_b200 as sp  # noqa: E402
from paper_1805_11938_b200 import dist as spdist, synth  # noqa: E402
from paper_1805_11938_b200.relabel import DegreeOrder  # noqa: E402


def report(name, m):
    c = m.c
    w = m.widths
    n_sl = w.numel()
    rows = torch.full((n_sl,), c, dtype=torch.int64, device=w.device)
    if m.n_rows % c:
        rows[-1] = m.n_rows % c
    cells = w * rows
    rn = m.row_nnz_perm.to(torch.int64)
    pad = torch.zeros(n_sl * c, dtype=torch.int64, device=w.device)
    pad[: rn.numel()] = rn
    nnz_sl = pad.view(n_sl, c).sum(1)
    wc = m.wide_cols()
    lst, n_wide, _, first, n_pieces, _, _, hub, n_hub = m.wide_plan()
    wide = w > wc
    line = [f"{name}: rows {m.n_rows} nnz {int(rn.sum())} cells {int(cells.sum())} "
            f"({int(cells.sum()) / max(int(rn.sum()), 1):.3f} x); wide_cols {wc}"]
    line.append(f"  wide slices {int(wide.sum())}: cells {int(cells[wide].sum())} nnz {int(nnz_sl[wide].sum())} "
                f"({int(cells[wide].sum()) / max(int(nnz_sl[wide].sum()), 1):.3f} x), pieces {n_pieces}")
    if n_hub:
        hs = lst[hub[:n_hub].long()].long()
        line.append(f"  hub slices {n_hub}: cells {int(cells[hs].sum())} nnz {int(nnz_sl[hs].sum())} "
                    f"({int(cells[hs].sum()) / max(int(nnz_sl[hs].sum()), 1):.3f} x)")
    nar = ~wide
    line.append(f"  narrow slices {int(nar.sum())}: cells {int(cells[nar].sum())} nnz {int(nnz_sl[nar].sum())}")
    print("\n".join(line), flush=True)


def main():
    dev = torch.device("cuda", 0)
    for wl in ("C4", "C5"):
        w = bench.WORKLOADS[wl]
        csr = sp.to_csr(bench.build_workload(sp, synth, w, dev))
        kw = dict(sell_c=32, sell_sigma=0, max_cells=1 << 34)
        order = DegreeOrder(csr)
        report(f"{wl} whole", sp.convert("sell", order.matrix(csr), **kw))
        torch.cuda.empty_cache()
        if wl == "C5":
            for P in (2, 4, 8):
                o = DegreeOrder(csr, parts=P)
                mat = o.matrix(csr)
                report(f"{wl} dealt shard 0/{P}", sp.convert("sell", spdist.row_block(mat, 0, o.part_bounds[1]), **kw))
                del mat, o
                torch.cuda.empty_cache()
        del csr, order
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
