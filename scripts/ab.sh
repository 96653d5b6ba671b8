#!/bin/bash
# A/B of kernel variants on C2-C4 (+C5 csr/csr5): prints one line per run.
for v in plain tma; do
  SPMVB_MERGE_KERNEL=$v SPMVB_CSR5_KERNEL=$v python scripts/bench_formats.py --configs ${CONFIGS:-C2,C3,C4} --reps 10 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l)
    if d['format'] in ('csr','csr5','hyb') and 'error' not in d:
        print('$v', d['config'], d['format'], d['variant'][:14], '%.1f us %.0f GB/s %.1f GF' % (d['cold_us'], d['gbs_model'], d['gflops']), d['within_tol'])
"
done
