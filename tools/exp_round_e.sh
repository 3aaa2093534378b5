# experiment E: early batch uploads (ring slots carved out of the planned reservation) vs after the setup
cd $GRAFT_REPO_ROOT
o=gpurun_out
timeout 900 python -m pytest -x -q tests/test_gpu_pipeline.py tests/test_gpu_ntt_chunked.py > $o/e_tests.log 2>&1
echo "tests rc=$?" > $o/e_early.txt
for cfg in "1 4" "0 2" "1 3" "1 4" "0 2"; do
  set -- $cfg
  echo "== HG_STREAM_EARLY=$1 HG_STREAM_SLOTS=$2" >> $o/e_early.txt
  HG_BENCH_DEBUG=1 HG_STREAM_EARLY=$1 HG_STREAM_SLOTS=$2 timeout 600 python bench.py --steps 3 --warmup 3 --no-primitives --no-cpu-baseline 2>> $o/e_early.txt | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['whole_job'], d['config0_job']['value'])" >> $o/e_early.txt 2>&1
done
