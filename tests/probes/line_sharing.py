"""Distinct 128-byte x lines touched by one 32-lane gather instruction for an
R-MAT matrix under three lane layouts (striped, 8 per lane, CSR5 sigma=16),
with original and degree-relabelled columns.  python tests/probes/line_sharing.py 21 10"""
import numpy as np, sys
sys.path.insert(0, __import__('pathlib').Path(__file__).resolve().parents[2].as_posix())
from oracle import synth_ref
scale, ef = int(sys.argv[1]), int(sys.argv[2])
r, c, v = synth_ref.rmat(scale, ef, 104)
r = r.astype(np.int64); c = c.astype(np.int64)
n = 1 << scale
def relabel_map(cnt):
    order = np.argsort(-cnt, kind='stable')
    rank = np.empty(n, np.int64); rank[order] = np.arange(n)
    return rank
def stats(r, c, tag):
    o = np.lexsort((c, r)); rr = r[o]; cc = c[o]
    nnz = len(cc)
    line = cc >> 4
    # lane-contiguous stripes: instruction groups = 32 consecutive entries (striped) -> distinct (row,line)
    for W, lab in ((1, 'striped'), (8, 'lane8'), (16, 'csr5_s16')):
        m = nnz // 512 * 512
        key = (rr[:m] << 24) | line[:m]
        K = key.reshape(-1, 32, 512 // 32 // 1) if False else None
        # entries per chunk of 256/512: instruction u accesses entries base + lane*W + u (W=lane stride)
        if W == 1:
            g = key.reshape(-1, 32)
        else:
            g = key.reshape(-1, 32, W).transpose(0, 2, 1).reshape(-1, 32)
        g = np.sort(g, axis=1)
        distinct = 1 + (np.diff(g, axis=1) != 0).sum(axis=1)
        print(f"{tag:10s} {lab:9s} nnz={nnz} mean distinct lines / 32 lanes = {distinct.mean():.2f}")
stats(r, c, 'orig')
cnt = np.bincount(c, minlength=n)
rk = relabel_map(cnt)
stats(r, rk[c], 'relabel')
