# experiment F: ring started before the M_dup ladders (default) vs with the setup vs after it
cd $GRAFT_REPO_ROOT
o=gpurun_out
timeout 900 python -m pytest -x -q tests/test_gpu_pipeline.py > $o/f_tests.log 2>&1
echo "tests rc=$?" > $o/f_early.txt
for cfg in "1 4 dup" "0 2 dup" "1 3 dup" "1 5 dup" "1 4 dup" "0 2 dup"; do
  set -- $cfg
  echo "== HG_STREAM_EARLY=$1 HG_STREAM_SLOTS=$2 HG_STREAM_WHEN=$3" >> $o/f_early.txt
  HG_BENCH_DEBUG=1 HG_STREAM_EARLY=$1 HG_STREAM_SLOTS=$2 HG_STREAM_WHEN=$3 timeout 600 python bench.py --steps 3 --warmup 3 --no-primitives --no-cpu-baseline 2>> $o/f_early.txt | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); w=d['whole_job']; print(d['value'], d['e2e']['value'], w['setup_s'], w['measured_s'], w['value'], d['config0_job']['value'])" >> $o/f_early.txt 2>&1
done
