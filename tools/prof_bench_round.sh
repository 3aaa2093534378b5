# the default bench line + the step's ncu launch list (cold-cache serialised) for profiles/
#   bash tools/prof_bench_round.sh <tag>
cd $GRAFT_REPO_ROOT
tag=$1
timeout 900 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
HG_PROFILE_STEP=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/${tag}_step_launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-primitives --no-cpu-baseline > gpurun_out/${tag}_ncu_step.log 2>&1
