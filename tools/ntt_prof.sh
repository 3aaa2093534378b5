cd $GRAFT_REPO_ROOT
timeout 300 python tools/ntt_bench.py > gpurun_out/ntt_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -o gpurun_out/ntt_c8 python tools/ntt_bench.py --ncu > gpurun_out/ntt_ncu.log 2>&1
