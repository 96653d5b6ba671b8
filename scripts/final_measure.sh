#!/bin/bash
# Round-end measurement set (one GPU): tests, bench (default + C5 format sweep),
# per-config format table, conversions, launch list of the default bench
# command and one full ncu capture of the headline kernel.
set -u
O=gpurun_out
python -m pytest tests -q -m gpu > $O/final_tests.log 2>&1
python bench.py > $O/final_bench.json 2> $O/final_bench.err
for w in C1 C2 C3 C4; do python bench.py --workload $w > $O/final_bench_$w.json 2> $O/final_bench_$w.err; done
python bench.py --formats csr,csr5,hyb,sell,ell --no-cpu-baseline > $O/final_bench_sweep.json 2> $O/final_sweep.err
python scripts/bench_formats.py --configs C1,C2,C3,C4 --reps 10 > $O/final_formats.jsonl 2> $O/final_formats.err
python scripts/bench_convert.py --configs C1,C2,C3,C4,C5 > $O/final_convert.jsonl 2> $O/final_convert.err
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 800 --csv \
  --log-file $O/final_launches_bench.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $O/final_ncu_launch.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_csr5_warp_s -s 3 -c 1 -o $O/r01_ncu_c5_csr5_final \
  python scripts/profile_kernel.py --workload C5 --format csr5 --reps 2 > $O/final_ncu_full.log 2>&1
