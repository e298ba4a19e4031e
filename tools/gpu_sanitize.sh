#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_driver.py
#   gpurun --timeout 2400 -- bash tools/gpu_sanitize.sh TAG
set -u
TAG=${1:-r2}
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_san_$TAG.log 2>&1
python tools/sanitize_driver.py > $OUT/san_plain_$TAG.log 2>&1; echo "plain rc=$?"
for tool in memcheck synccheck racecheck; do
  extra=""
  [ $tool = racecheck ] && extra="--racecheck-report hazard"
  timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool $tool $extra --print-limit 200 \
      python tools/sanitize_driver.py > $OUT/san_${tool}_$TAG.log 2>&1
  echo "$tool rc=$?"; tail -4 $OUT/san_${tool}_$TAG.log
done
