#!/bin/bash
# One measurement session for profiles/: GPU tests, smoke, the default bench (C2, with e2e and
# cpu_baseline), the other configs, the ncu launch list of the C2 step, ncu --set full of
# the dominant kernels (C2) and of the C4 hub kernel.
#   gpurun --timeout 3600 -- bash tools/gpu_round.sh TAG
set -u
TAG=${1:-r2}
OUT=gpurun_out; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $OUT/gpu_$TAG.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_$TAG.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu_$TAG.log
tail -3 $OUT/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke_$TAG.log
tail -2 $OUT/smoke_$TAG.log
timeout 900 python bench.py --kernel-table > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench rc=$?"
cat $OUT/bench_$TAG.json | cut -c1-400; head -12 $OUT/bench_$TAG.err
# the host-buffer path's per-block timeline (KK_HOST_TRACE=1) of one C2 call
KK_HOST_TRACE=1 timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2> $OUT/e2e_trace_$TAG.err
grep "kk host" $OUT/e2e_trace_$TAG.err | tail -40 > $OUT/e2e_trace_$TAG.txt
for C in C3 C3J C5 C4; do
  timeout 1200 python bench.py --config $C --steps 5 --warmup 3 --kernel-table --no-cpu-baseline > $OUT/bench_${C}_$TAG.json 2> $OUT/bench_${C}_$TAG.err
  echo "bench $C rc=$?"; cut -c1-300 $OUT/bench_${C}_$TAG.json; head -6 $OUT/bench_${C}_$TAG.err
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $OUT/launches_$TAG.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/ncu_launch_bench_$TAG.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k regex:"num_rank<int, double, \(int\)128,|sym_rows<int, \(int\)49152, \(int\)0" -s 2 -c 2 \
    -o /tmp/prof_top_$TAG -f python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/ncu_full_$TAG.log 2>&1; echo "ncu full rc=$?"
ncu -i /tmp/prof_top_$TAG.ncu-rep --page raw --csv > $OUT/raw_top_$TAG.csv 2>/dev/null
ncu -i /tmp/prof_top_$TAG.ncu-rep --page source --csv --print-source sass > $OUT/sass_top_$TAG.csv 2>/dev/null
gzip -c /tmp/prof_top_$TAG.ncu-rep > $OUT/prof_top_$TAG.ncu-rep.gz
timeout 900 ncu --set full --clock-control none --kernel-name-base demangled -k regex:"k_num_hub" -s 0 -c 1 \
    -o /tmp/prof_hub_$TAG -f python bench.py --config C4 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > $OUT/ncu_hub_$TAG.log 2>&1; echo "ncu hub rc=$?"
ncu -i /tmp/prof_hub_$TAG.ncu-rep --page raw --csv > $OUT/raw_hub_$TAG.csv 2>/dev/null
# the C4 side-stream strict tier and the C5 wide-pattern rank tier (one launch each)
timeout 900 ncu --set full --clock-control none --kernel-name-base demangled -k regex:"k_num_strict<long, double, \(int\)1024" -s 0 -c 1 \
    -o /tmp/prof_strict_$TAG -f python bench.py --config C4 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > $OUT/ncu_strict_$TAG.log 2>&1; echo "ncu strict rc=$?"
ncu -i /tmp/prof_strict_$TAG.ncu-rep --page raw --csv > $OUT/raw_strict_$TAG.csv 2>/dev/null
timeout 1200 ncu --set full --clock-control none --kernel-name-base demangled -k regex:"k_num_rank<long, double, \(int\)512" -s 0 -c 1 \
    -o /tmp/prof_rankh_$TAG -f python bench.py --config C5 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > $OUT/ncu_rankh_$TAG.log 2>&1; echo "ncu rank_hash rc=$?"
ncu -i /tmp/prof_rankh_$TAG.ncu-rep --page raw --csv > $OUT/raw_rankh_$TAG.csv 2>/dev/null
ls -la $OUT | tail -30
