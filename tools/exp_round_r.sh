# ring allocated behind the M_dup stage (HEAD) -- repeated runs, with and without the cyclic GC
cd $GRAFT_REPO_ROOT
o=gpurun_out
timeout 600 python -m pytest -x -q tests/test_gpu_pipeline.py > $o/r_tests.log 2>&1
echo "tests rc=$?" > $o/r_runs.txt
for gc in 0 1 0 1; do
  HG_BENCH_NOGC=$gc HG_BENCH_DEBUG=1 timeout 600 python bench.py --steps 2 --warmup 3 --no-primitives --no-cpu-baseline 2> $o/r_err.txt | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); w=d['whole_job']; print('nogc=$gc', 'setup', w['setup_s'], 'job', w['measured_s'], w['value'], 'config0', d['config0_job']['value'], 'e2e', d['e2e']['value'])" >> $o/r_runs.txt 2>&1
  grep "batch ms" $o/r_err.txt | cut -c1-260 >> $o/r_runs.txt
done
