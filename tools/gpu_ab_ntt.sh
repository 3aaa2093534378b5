# cluster NTT: parity tests, then same-box A/B of the batch step (two-pass vs cluster NTT)
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest -x -q tests/test_gpu_ntt_cluster.py > gpurun_out/ab_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ab_tests.log
timeout 900 python -m pytest -x -q tests/test_gpu_ring.py tests/test_gpu_scale_parity.py tests/test_gpu_fused.py >> gpurun_out/ab_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ab_tests.log
for v in 0 1 0 1; do HG_NTT_CLUSTER=$v timeout 400 python bench.py --steps 5 --warmup 3 --no-e2e --no-primitives --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cluster=$v', d['value'], d['ms_per_step'], json.dumps(d['roofline']['kernel_classes']))" >> gpurun_out/ab_bench.log 2>&1; done
