set -u
python -m paper_2103_11991_b200.build >/dev/null 2>&1
run() { # label dir config env...
  local lab=$1 dir=$2 cfg=$3; shift 3
  (cd $dir && env "$@" timeout 600 python bench.py --config $cfg --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --kernel-table > /tmp/o.json 2> /tmp/o.err)
  python -c "import json; d=json.loads(open('/tmp/o.json').read().strip().splitlines()[-1]); print('$lab', d['ms_per_step'], d['phases_ms']['symbolic'], d['phases_ms']['numeric'])"
  grep -E "num_rank_hash_S512|num_hub |num_tiny" /tmp/o.err | head -2
}
run C5_old .abtree C5 X=1
run C5_new . C5 X=1
run C4_new . C4 X=1
run C4_dyn . C4 KK_HUB_DYN=1
run C4_g74 . C4 KK_HUB_GRID=74
run C4_g100 . C4 KK_HUB_GRID=100
