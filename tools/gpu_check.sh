#!/bin/bash
# One gpurun session: parity tests, smoke, bench, ncu launch list and one full capture.
#   gpurun --timeout 2400 -- bash tools/gpu_check.sh [tag]
set -u
TAG=${1:-r1}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $OUT/gpu_$TAG.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_$TAG.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu_$TAG.log
tail -3 $OUT/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke_$TAG.log
tail -2 $OUT/smoke_$TAG.log
timeout 600 python bench.py --kernel-table > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench rc=$?"
cat $OUT/bench_$TAG.json; tail -30 $OUT/bench_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $OUT/launches_$TAG.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/ncu_launch_bench_$TAG.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k regex:"num_rank<int, double, \(int\)128,|sym_rows<int, \(int\)49152, \(int\)0" -s 2 -c 2 \
    -o /tmp/prof_top_$TAG -f python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/ncu_full_$TAG.log 2>&1; echo "ncu full rc=$?"
ncu -i /tmp/prof_top_$TAG.ncu-rep --page raw --csv > $OUT/raw_top_$TAG.csv 2>/dev/null
ncu -i /tmp/prof_top_$TAG.ncu-rep --page source --csv --print-source sass > $OUT/sass_top_$TAG.csv 2>/dev/null
gzip -c /tmp/prof_top_$TAG.ncu-rep > $OUT/prof_top_$TAG.ncu-rep.gz
ls -la $OUT
