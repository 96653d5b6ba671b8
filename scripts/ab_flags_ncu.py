"""ncu helper: C5 CSR5 SpMV with packed (arg 'packed') or byte flags."""
import sys
import torch
sys.path.insert(0, '.')
import paper_1805_11938_b200 as sp
from paper_1805_11938_b200 import synth, kernels
dev = torch.device('cuda', 0)
r, c, v = synth.rmat_triplets(25, 16, 105, dev)
n = 1 << 25
m = sp.to_csr5(sp.to_csr(sp.canonicalize(r, c, v, n, n)), 32, 16)
del r, c, v
x = synth.uniform_vector(n, 7, device=dev)
y = torch.empty(n, dtype=torch.float64, device=dev)
if sys.argv[1] != 'packed':
    kernels._PACKED_FLAGS_MIN_X_BYTES = 1 << 62
for _ in range(5):
    sp.spmv('csr5', m, x, out=y)
torch.cuda.synchronize()
