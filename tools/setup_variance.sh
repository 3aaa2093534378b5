for conf in "" "expandable_segments:True"; do
  for i in 1 2 3; do
    PYTORCH_CUDA_ALLOC_CONF=$conf timeout 700 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-primitives --no-e2e > gpurun_out/b_$i.log 2>&1
    python - "$conf" gpurun_out/b_$i.log <<'PY'
import json, sys
line = open(sys.argv[2]).read().strip().splitlines()[-1]
d = json.loads(line)
print(repr(sys.argv[1]), d["ms_per_step"], d["whole_job"]["setup_s"], d["whole_job"]["value"])
PY
  done
done
