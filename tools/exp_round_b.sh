# experiments batch B: ncu --set full of the batch step's unit of work (four prepared products), new probe
cd $GRAFT_REPO_ROOT
o=gpurun_out
timeout 300 python tools/profile_one.py --op mult4 > $o/b_plain.log 2>&1 || exit 1
timeout 1200 ncu --set full --clock-control none --import-source on --profile-from-start off -o $o/b_mult4_full -f python tools/profile_one.py --op mult4 > $o/b_ncu.log 2>&1
timeout 400 python bench.py --steps 5 --warmup 3 --no-e2e --no-primitives --no-cpu-baseline 2>/dev/null | tail -1 > $o/b_bench.json
