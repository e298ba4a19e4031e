#!/bin/bash
# Quick gpurun iteration: build, GPU parity tests (optional filter), bench, optional ncu of one kernel.
#   gpurun -- bash tools/gpu_quick.sh TAG [pytest -k expr|all|none] [ncu kernel regex|none] [bench args...]
set -u
TAG=$1; KEXPR=${2:-all}; NCUK=${3:-none}; shift 3 || true
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_$TAG.log 2>&1 || { echo BUILD FAILED; tail $OUT/build_$TAG.log; }
if [ "$KEXPR" != "none" ]; then
  if [ "$KEXPR" = "all" ]; then timeout 1200 python -m pytest tests -m gpu -q > $OUT/pytest_$TAG.log 2>&1
  else timeout 900 python -m pytest tests -m gpu -x -q -k "$KEXPR" > $OUT/pytest_$TAG.log 2>&1; fi
  echo "pytest rc=$?"; tail -15 $OUT/pytest_$TAG.log
fi
timeout 600 python bench.py --kernel-table --no-e2e --no-cpu-baseline "$@" > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench rc=$?"
cat $OUT/bench_$TAG.json; tail -25 $OUT/bench_$TAG.err
if [ "$NCUK" != "none" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"$NCUK" -s 1 -c 2 \
      -o /tmp/prof_$TAG -f python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline "$@" > $OUT/ncu_$TAG.log 2>&1; echo "ncu rc=$?"
  ncu -i /tmp/prof_$TAG.ncu-rep --page raw --csv > $OUT/raw_$TAG.csv 2>/dev/null
  ncu -i /tmp/prof_$TAG.ncu-rep --page source --csv --print-source sass > $OUT/sass_$TAG.csv 2>/dev/null
  gzip -c /tmp/prof_$TAG.ncu-rep > $OUT/prof_$TAG.ncu-rep.gz
fi
