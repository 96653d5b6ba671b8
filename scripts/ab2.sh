#!/bin/bash
# A/B: CSR/HYB merge-path vs chunked (S=16 / S=8) on C1-C4
for v in merge chunk16 chunk8; do
  case $v in merge) export SPMVB_CSR_KERNEL=merge;; chunk16) export SPMVB_CSR_KERNEL=chunk SPMVB_CSR_CHUNK_S=16;; chunk8) export SPMVB_CSR_KERNEL=chunk SPMVB_CSR_CHUNK_S=8;; esac
  python scripts/bench_formats.py --configs ${CONFIGS:-C1,C2,C3,C4} --reps 10 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l)
    if d['format'] in ('csr','hyb') and 'error' not in d:
        print('$v', d['config'], d['format'], '%8.1f us %6.0f GB/s %7.1f GF | hot %7.1f GF' % (d['cold_us'], d['gbs_model'], d['gflops'], d['hot_gflops']), d['within_tol'])
"
done
