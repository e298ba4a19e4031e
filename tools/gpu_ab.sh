#!/bin/bash
# A/B kernel variants on one box: build, optional GPU tests, then bench.py once per env setting.
#   gpurun -- bash tools/gpu_ab.sh TAG "pytest -k expr|all|none" "ENV1=a ENV2=b" "ENV1=c" ...
# Each bench line goes to gpurun_out/ab_TAG.txt prefixed by its env setting.
set -u
TAG=$1; KEXPR=$2; shift 2
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_$TAG.log 2>&1 || { echo BUILD FAILED; tail $OUT/build_$TAG.log; }
if [ "$KEXPR" != "none" ]; then
  if [ "$KEXPR" = "all" ]; then timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_$TAG.log 2>&1
  else timeout 900 python -m pytest tests -m gpu -x -q -k "$KEXPR" > $OUT/pytest_$TAG.log 2>&1; fi
  echo "pytest rc=$?"; tail -15 $OUT/pytest_$TAG.log
fi
: > $OUT/ab_$TAG.txt
for SETTING in "$@"; do
  echo "=== $SETTING" | tee -a $OUT/ab_$TAG.txt
  env $SETTING timeout 600 python bench.py --kernel-table --no-e2e --no-cpu-baseline ${BENCH_ARGS:-} > $OUT/ab_one.json 2> $OUT/ab_one.err
  echo "rc=$?" >> $OUT/ab_$TAG.txt
  python -c "import json;d=json.load(open('$OUT/ab_one.json'));print('ms/step',d['ms_per_step'],'GFLOP/s',d['value'],'phases',d['phases_ms'],'num frac',d['roofline']['frac'])" | tee -a $OUT/ab_$TAG.txt
  head -8 $OUT/ab_one.err | tee -a $OUT/ab_$TAG.txt
done
