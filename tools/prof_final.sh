# launch list of one batch step + ncu --set full of the batch unit's top kernels (mult4)
cd $GRAFT_REPO_ROOT
tag=$1
HG_PROFILE_STEP=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/${tag}_step_launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-primitives --no-cpu-baseline > gpurun_out/${tag}_ncu_step.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on --profile-from-start off -c 16 -o gpurun_out/${tag}_mult4_full python tools/profile_one.py --op mult4 > gpurun_out/${tag}_ncu_full.log 2>&1
