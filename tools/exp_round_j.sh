# A/B of the batch ring on one box, alternating: slots 4 / 3 from the M_dup stage, and 2 slots after the setup
cd $GRAFT_REPO_ROOT
o=gpurun_out
: > $o/j_slots.txt
for rep in 1 2 3; do
for cfg in "1 4" "1 3" "0 2"; do
  set -- $cfg
  HG_BENCH_DEBUG=1 HG_STREAM_EARLY=$1 HG_STREAM_SLOTS=$2 timeout 600 python bench.py --steps 2 --warmup 3 --no-primitives --no-cpu-baseline 2> $o/j_err.txt | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); w=d['whole_job']; print('early=$1 slots=$2', 'setup', w['setup_s'], 'job', w['measured_s'], w['value'], 'config0', d['config0_job']['value'])" >> $o/j_slots.txt 2>&1
  grep "batch ms" $o/j_err.txt | cut -c1-260 >> $o/j_slots.txt
done
done
