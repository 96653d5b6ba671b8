#!/bin/bash
# Round-end measurement set (one GPU): tests, smoke, both bench arms, the
# --workload lines, per-config format table, conversions, Matrix Market I/O,
# the ncu launch list of the default bench command, the DRAM traffic of every
# reported kernel and one full ncu capture of the headline kernels (C5
# degree-ordered SELL-32).  Everything lands in gpurun_out/ with prefix $P.
#   bash scripts/final_measure.sh [prefix]
set -u
P=${1:-final}
O=gpurun_out
mkdir -p $O
python -m pytest tests -q -m gpu > $O/${P}_tests.log 2>&1
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/${P}_smoke.log 2>&1
python bench.py --impl reference --steps 3 --warmup 1 > $O/${P}_ref.json 2> $O/${P}_ref.err
python bench.py > $O/${P}_bench.json 2> $O/${P}_bench.err
for w in C1 C2 C3 C4; do python bench.py --workload $w --no-cpu-baseline > $O/${P}_bench_$w.json 2> $O/${P}_bench_$w.err; done
python scripts/bench_formats.py --configs C1,C2,C3,C4 --reps 10 > $O/${P}_formats.jsonl 2> $O/${P}_formats.err
python scripts/bench_convert.py --configs C1,C2,C3,C4,C5 > $O/${P}_convert.jsonl 2> $O/${P}_convert.err
python scripts/mm_io_bench.py > $O/${P}_mm_io.txt 2>&1
# after the plain runs have exited 0: the launch list of the same bench command
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 1500 --csv \
  --log-file $O/${P}_launches_bench.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-configs \
  > $O/${P}_ncu_launch.log 2>&1
ncu --set full --import-source on --clock-control none -k "regex:k_spmv_sell|k_sell_wide_part" -s 6 -c 2 \
  -o $O/${P}_ncu_c5_sell python scripts/profile_kernel.py --workload C5 --format sell --relabel --reps 2 \
  > $O/${P}_ncu_full.log 2>&1
ncu -i $O/${P}_ncu_c5_sell.ncu-rep --page raw --csv > $O/${P}_ncu_c5_sell_raw.csv 2>/dev/null
tail -3 $O/${P}_tests.log
cat $O/${P}_smoke.log | tail -1
