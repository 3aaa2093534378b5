# A/B of library builds on one box: parity tests on each candidate, then the batch step
#   bash tools/gpu_ab_libs.sh <tag> <lib> [<lib> ...]   (lib "main" = the in-tree build)
cd $GRAFT_REPO_ROOT
tag=$1; shift
for lib in "$@"; do
  if [ "$lib" = main ]; then unset HG_LIB_PATH; else export HG_LIB_PATH=$lib; fi
  timeout 900 python -m pytest -x -q tests/test_gpu_ring.py tests/test_gpu_scale_parity.py tests/test_gpu_fused.py tests/test_gpu_ckks.py tests/test_gpu_pipeline.py tests/test_gpu_batched_ops.py > gpurun_out/${tag}_tests_$(basename $(dirname $lib)).log 2>&1
  echo "$lib tests rc=$?" >> gpurun_out/${tag}_ab.log
done
for rep in 1 2; do
  for lib in "$@"; do
    if [ "$lib" = main ]; then unset HG_LIB_PATH; else export HG_LIB_PATH=$lib; fi
    timeout 400 python bench.py --steps 5 --warmup 3 --no-e2e --no-primitives --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['roofline']['kernel_classes']; print('$lib', d['value'], d['ms_per_step'], {c: k[c]['ms_per_step'] for c in k})" >> gpurun_out/${tag}_ab.log 2>&1
  done
done
