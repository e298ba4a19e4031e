#!/bin/bash
# ncu --set full of kernels matching a regex in the bench (one launch each after warm-up);
# exports the raw and source (cuda,sass) pages as CSV on the box, keeps the .ncu-rep gzipped.
#   gpurun -- bash tools/gpu_ncu.sh TAG "regex" [bench args...]
set -u
TAG=$1; RE=$2; shift 2
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"$RE" -s 2 -c ${NCU_COUNT:-2} \
    -o /tmp/prof_$TAG -f python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline "$@" > $OUT/ncu_$TAG.log 2>&1; echo "ncu rc=$?"
tail -3 $OUT/ncu_$TAG.log
ncu -i /tmp/prof_$TAG.ncu-rep --page raw --csv > $OUT/raw_$TAG.csv 2>/dev/null
ncu -i /tmp/prof_$TAG.ncu-rep --page source --csv --print-source cuda,sass > $OUT/src_$TAG.csv 2>/dev/null
gzip -c /tmp/prof_$TAG.ncu-rep > $OUT/prof_$TAG.ncu-rep.gz
ls -la $OUT/*_$TAG*
