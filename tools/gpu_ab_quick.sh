# quick same-box A/B of library builds (no parity tests: run them on the winner): batch step, 2 rounds
#   bash tools/gpu_ab_quick.sh <tag> <lib> [<lib> ...]   (lib "main" = the in-tree build)
cd $GRAFT_REPO_ROOT
tag=$1; shift
for rep in 1 2; do
  for lib in "$@"; do
    if [ "$lib" = main ]; then unset HG_LIB_PATH; else export HG_LIB_PATH=$lib; fi
    timeout 400 python bench.py --steps 5 --warmup 3 --no-e2e --no-primitives --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['roofline']['kernel_classes']; print('$lib', d['value'], d['ms_per_step'], {c: k[c]['ms_per_step'] for c in k}, d['clocks']['sm_mhz'])" >> gpurun_out/${tag}_ab.log 2>&1
  done
done
