#!/bin/bash
# A/B of an environment switch on one box: bench once per value.
#   gpurun -- bash tools/gpu_ab_env.sh TAG VAR "v1 v2 ..." [bench args...]
set -u
TAG=$1; VAR=$2; VALS=$3; shift 3
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_$TAG.log 2>&1
for v in $VALS; do
  env $VAR=$v timeout 900 python bench.py --kernel-table --no-e2e --no-cpu-baseline "$@" > $OUT/ab_${TAG}_$v.json 2> $OUT/ab_${TAG}_$v.err
  echo "== $VAR=$v rc=$?"; python -c "import json;d=json.load(open('$OUT/ab_${TAG}_$v.json'));print(d['ms_per_step'], d['phases_ms'])"
  grep -E "^  (num_|sym_)" $OUT/ab_${TAG}_$v.err | head -4
done
