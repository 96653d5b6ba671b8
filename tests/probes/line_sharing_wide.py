"""Distinct 128-byte x lines per 32-lane gather for the rows of the wide SELL
slices of the degree-ordered R-MAT matrix, under two traversals: 32 rows at
one slot (the current k_sell_wide_part) and one row at 32 consecutive slots.
    python tests/probes/line_sharing_wide.py 21 10 104 > profiles/r02_line_sharing_wide.txt"""
import sys, numpy as np
sys.path.insert(0, __import__('pathlib').Path(__file__).resolve().parents[2].as_posix())
from oracle import cpu_baseline
scale, ef, seed = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
ptr, ind, dat = cpu_baseline.rmat_full_csr(scale, ef, seed)
n = 1 << scale
rowdeg = np.diff(ptr); coldeg = np.bincount(ind, minlength=n)
perm = np.lexsort((np.arange(n), -coldeg, -rowdeg, rowdeg == 0))
new = np.empty(n, np.int64); new[perm] = np.arange(n)
# relabelled rows in new order
for thr in (256, 4096):
    rows = perm[:np.sum(rowdeg > thr)]  # old ids of rows longer than thr, in new order
    rows = rows[: (rows.size // 32) * 32]
    tot_a = tot_b = cnt = 0
    for s in range(0, min(rows.size, 32 * 64), 32):
        sl = rows[s:s + 32]
        cols = [np.sort(new[ind[ptr[r]:ptr[r + 1]]]) for r in sl]
        w = min(len(c) for c in cols)
        w = (w // 32) * 32
        if w == 0: continue
        M = np.stack([c[:w] for c in cols]) >> 4  # line ids (16 doubles per 128 B)
        # (a) current: warp = 32 rows at slot j
        a = np.array([np.unique(M[:, j]).size for j in range(w)])
        # (b) transposed: warp = one row, 32 consecutive slots
        b = np.array([np.unique(M[r, j:j + 32]).size for r in range(32) for j in range(0, w, 32)])
        tot_a += a.mean(); tot_b += b.mean(); cnt += 1
    print(f"scale {scale}: rows > {thr}: {rows.size} rows; lines per 32-lane gather: rows-at-slot {tot_a/cnt:.2f}, "
          f"row-consecutive {tot_b/cnt:.2f} (first {cnt} slices)")
