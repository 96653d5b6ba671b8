#!/bin/bash
# A/B of an environment knob on the C5 CSR5 SpMV: ab_env.sh VAR v1 v2 ...
var=$1; shift
for t in 1 2; do for v in "$@"; do env $var=$v python - <<'PY'
import os, sys, torch
sys.path.insert(0, '.')
import paper_1805_11938_b200 as sp
from paper_1805_11938_b200 import synth
dev = torch.device('cuda', 0)
r, c, v = synth.rmat_triplets(25, 16, 105, dev)
n = 1 << 25
m = sp.to_csr5(sp.to_csr(sp.canonicalize(r, c, v, n, n)), 32, 16)
del r, c, v
x = synth.uniform_vector(n, 7, device=dev)
y = torch.empty(n, dtype=torch.float64, device=dev)
for _ in range(5): sp.spmv('csr5', m, x, out=y)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(30): sp.spmv('csr5', m, x, out=y)
b.record(); torch.cuda.synchronize()
print(sys.argv, {k: os.environ[k] for k in os.environ if k.startswith('SPMVB_')}, round(a.elapsed_time(b)/30, 3), 'ms', flush=True)
PY
done; done
