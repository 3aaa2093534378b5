# L2-exchange cluster NTT: parity, microbenchmark, batch-step A/B (variant 0 vs 2)
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest -x -q tests/test_gpu_ntt_cluster.py > gpurun_out/v2_tests.log 2>&1; echo "rc=$?" >> gpurun_out/v2_tests.log
timeout 300 python tools/ntt_bench.py --variants 0 2 0 2 > gpurun_out/v2_nttbench.log 2>&1
for v in 0 2 0 2; do HG_NTT_CLUSTER=$v timeout 400 python bench.py --steps 5 --warmup 3 --no-e2e --no-primitives --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['roofline']['kernel_classes']; print('variant=$v', d['value'], d['ms_per_step'], {c: k[c]['ms_per_step'] for c in k})" >> gpurun_out/v2_bench.log 2>&1; done
