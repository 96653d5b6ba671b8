"""Wall time of canonicalize (the public call: plan, sort, sums, emit) on the
R-MAT configs, for same-box A/B runs between library builds (SPMVB_LIB_PATH)."""
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_1805_11938_b200 as sp  # noqa: E402
from paper_1805_11938_b200 import synth  # noqa: E402

tag = Path(os.environ.get("SPMVB_LIB_PATH", "working-tree")).name
for scale, ef, seed in [(21, 10, 104), (25, 16, 105)]:
    r, c, v = synth.rmat_triplets(scale, ef, seed, torch.device("cuda", 0))
    ts = []
    for _ in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        a = sp.canonicalize(r, c, v, 1 << scale, 1 << scale)
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
        del a
    print(f"{tag:22s} scale {scale}: canonicalize ms {' '.join(f'{t:.1f}' for t in ts)}", flush=True)
    del r, c, v
    torch.cuda.empty_cache()
