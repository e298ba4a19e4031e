set -u
python -m paper_2103_11991_b200.build >/dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "C2 or window_and_pattern or jacobi or deterministic" 2>&1 | tail -2
run() { local lab=$1 dir=$2 cfg=$3; shift 3
  (cd $dir && env "$@" timeout 600 python bench.py --config $cfg --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --kernel-table > /tmp/o.json 2> /tmp/o.err)
  python -c "import json; d=json.loads(open('/tmp/o.json').read().strip().splitlines()[-1]); print('$lab', d['ms_per_step'], d['phases_ms']['symbolic'], d['phases_ms']['numeric'])"
  grep -E "num_rank" /tmp/o.err | head -1; }
run C2_old .abtree C2 X=1
run C2_new . C2 X=1
run C2_old .abtree C2 X=1
run C2_new . C2 X=1
