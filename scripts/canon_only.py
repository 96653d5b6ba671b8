import sys, torch
sys.path.insert(0, '.')
import paper_1805_11938_b200 as sp
from paper_1805_11938_b200 import synth
r, c, v = synth.rmat_triplets(25, 16, 105, torch.device('cuda', 0))
for _ in range(2):
    a = sp.canonicalize(r, c, v, 1 << 25, 1 << 25)
    torch.cuda.synchronize()
