set -x
cd $GRAFT_REPO_ROOT
timeout 600 python tools/setup_cold.py > gpurun_out/r2_setup_cold.txt 2>&1
HG_PROFILE_STEP=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2_step_launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-primitives --no-cpu-baseline > gpurun_out/r2_ncu_step.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -c 12 -o gpurun_out/r2_mult4_full python tools/profile_one.py --op mult4 > gpurun_out/r2_ncu_full.log 2>&1
ls -la gpurun_out
