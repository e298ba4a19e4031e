#!/bin/bash
# Full-size configs: benches for C3, C5, C4 and the opt-in full-size parity tests.
set -u
OUT=gpurun_out; TAG=${1:-r1u}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_$TAG.log 2>&1
for C in C3 C3J C5 C4; do
  timeout 1200 python bench.py --config $C --steps 5 --warmup 3 --kernel-table > $OUT/bench_${C}_$TAG.json 2> $OUT/bench_${C}_$TAG.err
  echo "bench $C rc=$?"; cat $OUT/bench_${C}_$TAG.json | cut -c1-600; tail -12 $OUT/bench_${C}_$TAG.err
done
KK_FULLSIZE=1 timeout 2400 python -m pytest tests/test_gpu_fullsize.py -m gpu -x -q > $OUT/pytest_full_$TAG.log 2>&1; echo "fullsize rc=$?"; tail -15 $OUT/pytest_full_$TAG.log
