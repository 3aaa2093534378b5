# alternating same-box A/B of the batch ring: early=1 (started before the M_dup ladders, N slots) vs early=0 (2 slots, after the setup)
#   bash tools/ab_ring.sh <tag> "<early> <slots>" ...
cd $GRAFT_REPO_ROOT
tag=$1; shift
cfgs=("$@")
o=gpurun_out
: > $o/${tag}_ring.txt
for rep in 1 2 3; do
for cfg in "${cfgs[@]}"; do
  set -- $cfg
  HG_BENCH_DEBUG=1 HG_STREAM_EARLY=$1 HG_STREAM_SLOTS=$2 timeout 600 python bench.py --steps 2 --warmup 3 --no-primitives --no-cpu-baseline 2> $o/${tag}_err.txt | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); w=d['whole_job']; print('early=$1 slots=$2', 'setup', w['setup_s'], 'job', w['measured_s'], w['value'], 'config0', d['config0_job']['value'], 'e2e', d['e2e']['value'])" >> $o/${tag}_ring.txt 2>&1
  grep "batch ms" $o/${tag}_err.txt | cut -c1-260 >> $o/${tag}_ring.txt
  tail -2 $o/${tag}_err.txt | grep -i -E "error|Traceback" >> $o/${tag}_ring.txt
done
done
