import sys, torch
sys.path.insert(0, '.')
import paper_1805_11938_b200 as sp
from paper_1805_11938_b200 import synth
dev = torch.device('cuda', 0)
scale, ef = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (25, 16)
r, c, v = synth.rmat_triplets(scale, ef, 105, dev)
n = 1 << scale
m = sp.to_csr5(sp.to_csr(sp.canonicalize(r, c, v, n, n)), 32, 16)
del r, c, v
x = synth.uniform_vector(n, 7, device=dev)
y = torch.empty(n, dtype=torch.float64, device=dev)
bits = m.flag_bits
def t(reps=20):
    for _ in range(3): sp.spmv('csr5', m, x, out=y)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): sp.spmv('csr5', m, x, out=y)
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
m.flag_bits = None; y0 = sp.spmv('csr5', m, x).clone()
m.flag_bits = bits; y1 = sp.spmv('csr5', m, x).clone()
print('identical', bool(torch.equal(y0, y1)))
for trial in range(3):
    m.flag_bits = bits; tb = t()
    m.flag_bits = None; tn = t()
    print(f"scale {scale}: packed flags {tb:.3f} ms   byte flags {tn:.3f} ms")
